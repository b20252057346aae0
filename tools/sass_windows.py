"""Instruction / stall-sample share of an ncu report's kernel by SASS address
window (finds the hot region of a kernel).  usage: sass_windows.py rep kernel_regex [win]"""
import collections, csv, io, subprocess, sys
rep, kre = sys.argv[1], sys.argv[2]
win = int(sys.argv[3], 0) if len(sys.argv) > 3 else 0x200
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kre}",
                      "--launch-count", "1", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
c = {k: i for i, k in enumerate(hdr)}
def f(r, k):
    try: return float(r[c[k]])
    except (ValueError, KeyError, IndexError): return 0.0
body, seen = [], set()
for r in rows[2:]:
    try: a = int(r[c["Address"]], 16)
    except ValueError: continue
    if a not in seen:
        seen.add(a); body.append((a, r))
base = min(a for a, _ in body)
ti = sum(f(r, "Instructions Executed") for _, r in body) or 1
ts = sum(f(r, "Warp Stall Sampling (All Samples)") for _, r in body) or 1
wi, ws, first = collections.Counter(), collections.Counter(), {}
for a, r in body:
    k = (a - base) // win
    wi[k] += f(r, "Instructions Executed"); ws[k] += f(r, "Warp Stall Sampling (All Samples)")
    first.setdefault(k, r[c["Source"]].strip()[:60])
print(f"insts {ti:.0f} samples {ts:.0f}")
for k in sorted(wi):
    if wi[k] > 0.01 * ti or ws[k] > 0.01 * ts:
        print(f"{k * win:#07x} inst {100 * wi[k] / ti:5.1f}%  stall {100 * ws[k] / ts:5.1f}%  {first[k]}")
