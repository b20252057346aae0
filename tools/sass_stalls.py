"""Per-SASS-line stall reasons of one kernel, in program order, for lines
with at least `min` samples.  usage: sass_stalls.py rep kernel_regex [min]"""
import csv, io, subprocess, sys
rep, kre = sys.argv[1], sys.argv[2]
mn = float(sys.argv[3]) if len(sys.argv) > 3 else 5
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kre}",
                      "--launch-count", "1", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
c = {k: i for i, k in enumerate(hdr)}
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
seen = set()
tot = 0
body = []
for r in rows[2:]:
    if len(r) < len(hdr) or r[0] == "Address" or r[c['Address']] in seen:
        continue
    seen.add(r[c['Address']])
    body.append(r)
    tot += float(r[c['Warp Stall Sampling (All Samples)']] or 0)
for r in body:
    s = float(r[c['Warp Stall Sampling (All Samples)']] or 0)
    if s < mn:
        continue
    top = sorted(((float(r[c[k]] or 0), k[6:]) for k in reasons), reverse=True)[:3]
    print(f"{100*s/tot:5.1f}% {int(float(r[c['Instructions Executed']] or 0)):8d} "
          f"{r[c['Source']].strip()[:60]:60s} " + " ".join(f"{k}={v:.0f}" for v, k in top if v))
