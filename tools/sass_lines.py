"""Stall samples and executed instructions of an ncu report's kernel per
CUDA source line: the report's per-SASS-address metrics joined with the
cubin's line table (nvdisasm -g).  usage: sass_lines.py rep kernel_regex obj.o [n]"""
import collections, csv, glob, io, os, re, subprocess, sys, tempfile

rep, kre, obj = sys.argv[1], sys.argv[2], sys.argv[3]
n = int(sys.argv[4]) if len(sys.argv) > 4 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kre}", "--launch-count", "1",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
c = {k: i for i, k in enumerate(hdr)}
base = None
samples, insts = {}, {}
for r in rows[2:]:
    if len(r) < len(hdr) or r[0] == "Address":
        continue
    a = int(r[c["Address"]], 16)
    base = a if base is None else min(base, a)
    samples[a] = float(r[c["Warp Stall Sampling (All Samples)"]] or 0)
    insts[a] = float(r[c["Instructions Executed"]] or 0)
with tempfile.TemporaryDirectory() as d:
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
    cubin = glob.glob(os.path.join(d, "*.cubin"))[0]
    dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
# the kernel's function section: find the function whose name matches kre
line_of = {}
cur_line, in_fn, fn_off = None, False, None
for ln in dis.splitlines():
    m = re.match(r"\s*\.text\.(\S+):", ln) or re.match(r"^(\S+):\s*$", ln)
    if ".text." in ln and ":" in ln and re.search(kre, ln):
        in_fn = True
        continue
    if in_fn and ln.startswith(".section") and ".text." in ln and not re.search(kre, ln):
        in_fn = False
    if not in_fn:
        continue
    m = re.search(r'line (\d+)', ln)
    if m and "//##" in ln:
        cur_line = int(m.group(1))
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/", ln)
    if m and cur_line is not None:
        line_of[int(m.group(1), 16)] = cur_line
agg_s, agg_i = collections.Counter(), collections.Counter()
for a, v in samples.items():
    l = line_of.get(a - base)
    agg_s[l] += v
    agg_i[l] += insts[a]
tot_s, tot_i = sum(agg_s.values()) or 1, sum(agg_i.values()) or 1
src = open(glob.glob(os.path.join(os.path.dirname(os.path.abspath(obj)), "..", "csrc", "*"))[0]).read() if False else None
print(f"lines mapped: {len(line_of)}; top lines by stall samples")
for l, v in agg_s.most_common(n):
    print(f"line {l}: stall {100 * v / tot_s:5.1f}%  inst {100 * agg_i[l] / tot_i:5.1f}%")
