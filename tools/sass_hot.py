"""Hottest SASS instructions of one kernel in an ncu report (stall samples and
executed instructions).  usage: sass_hot.py rep kernel_regex [n]"""
import csv, io, subprocess, sys
rep, kre = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kre}",
                      "--launch-count", "1", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
c = {k: i for i, k in enumerate(hdr)}
body = rows[2:]
def f(r, k):
    try: return float(r[c[k]])
    except (ValueError, KeyError, IndexError): return 0.0
tot_s = sum(f(r, "Warp Stall Sampling (All Samples)") for r in body) or 1
tot_i = sum(f(r, "Instructions Executed") for r in body) or 1
print(f"{rows[0][1][:100]}\n total samples {tot_s:.0f}, warp insts {tot_i:.0f}, sass lines {len(body)}")
if "--seq" in sys.argv:
    for r in body:
        print(f"{f(r,'Warp Stall Sampling (All Samples)'):7.0f} {f(r,'Instructions Executed'):9.0f}  {r[c['Source']].strip()[:90]}")
    sys.exit()
for r in sorted(body, key=lambda r: -f(r, "Warp Stall Sampling (All Samples)"))[:n]:
    print(f"{100*f(r,'Warp Stall Sampling (All Samples)')/tot_s:5.1f}% {f(r,'Instructions Executed'):9.0f}  {r[c['Address']][-5:]} {r[c['Source']].strip()[:90]}")
