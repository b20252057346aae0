"""Summarise an ncu report: per kernel duration, DRAM bytes, occupancy, top
stall reasons and hottest SASS lines.  usage: ncu_summary.py rep [regex]"""
import csv, io, re, subprocess, sys, collections

rep = sys.argv[1]
kre = sys.argv[2] if len(sys.argv) > 2 else "."
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units = rows[0], rows[1]
col = {k: i for i, k in enumerate(h)}
def g(r, k):
    i = col.get(k)
    return r[i] if i is not None else "?"
stall_cols = [k for k in h if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")]
seen = set()
for r in rows[2:]:
    name = g(r, "Kernel Name")
    if not re.search(kre, name) or name in seen:
        continue
    seen.add(name)
    print(f"== {name[:90]}")
    print(f"   dur={g(r,'gpu__time_duration.sum')}us dramR={g(r,'dram__bytes_read.sum')} dramW={g(r,'dram__bytes_write.sum')} "
          f"warps_active%={g(r,'sm__warps_active.avg.pct_of_peak_sustained_active')} "
          f"issue%={g(r,'sm__inst_issued.avg.pct_of_peak_sustained_active')} regs={g(r,'launch__registers_per_thread')} "
          f"grid={g(r,'launch__grid_size')} block={g(r,'launch__block_size')} inst={g(r,'smsp__inst_executed.sum')}")
    st = []
    for k in stall_cols:
        try:
            st.append((float(r[col[k]].replace(',', '')), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        except ValueError:
            pass
    tot = sum(v for v, _ in st) or 1
    print("   stalls:", ", ".join(f"{n}={100*v/tot:.0f}%" for v, n in sorted(st, reverse=True)[:6]))
