"""Group a kernel's SASS by execution count (one group ~ one code region).
usage: sass_groups.py rep kernel_regex [min_count_to_print_lines]"""
import csv, io, subprocess, sys, collections
rep, kre = sys.argv[1], sys.argv[2]
show = int(sys.argv[3]) if len(sys.argv) > 3 else 0
skip = sys.argv[4] if len(sys.argv) > 4 else "0"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kre}",
                      "--launch-skip", skip, "--launch-count", "1", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
c = {k: i for i, k in enumerate(hdr)}
seen, lst = set(), []
for r in rows[2:]:
    if len(r) < len(hdr) or r[0] == "Address" or r[c['Address']] in seen:
        continue
    seen.add(r[c['Address']])
    lst.append(r)
f = lambda r, k: float(r[c[k]] or 0)
agg, n, smp = collections.Counter(), collections.Counter(), collections.Counter()
for r in lst:
    ie = int(f(r, 'Instructions Executed'))
    agg[ie] += ie; n[ie] += 1; smp[ie] += f(r, 'Warp Stall Sampling (All Samples)')
tot, ts = sum(agg.values()), sum(smp.values())
print(f"total warp-inst {tot:.0f}  samples {ts:.0f}")
print(" count  n_inst  inst_total  %inst  %samples")
for k, v in sorted(agg.items(), key=lambda x: -x[1])[:16]:
    print(f"{k:7d} {n[k]:6d} {v:11.0f} {100*v/tot:5.1f} {100*smp[k]/ts:6.1f}")
if show:
    for r in lst:
        ie = int(f(r, 'Instructions Executed'))
        if ie == show:
            print(f"{f(r,'Warp Stall Sampling (All Samples)'):5.0f} {r[c['Source']].strip()[:90]}")
