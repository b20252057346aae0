#!/usr/bin/env bash
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/w5_launches.csv python tools/prof_cfg4.py > gpurun_out/w5_prof.out 2>&1
python - <<'PY'
import csv
lines = open("gpurun_out/w5_launches.csv").read().splitlines()
rows = list(csv.DictReader(lines[[i for i, l in enumerate(lines) if l.startswith("\"ID\"")][0]:]))
agg = {}
for r in rows:
    k = (r["ID"], r["Kernel Name"][:60])
    agg.setdefault(k, {})[r["Metric Name"]] = r["Metric Value"]
for (i, n), m in agg.items():
    print(i, n, m.get("gpu__time_duration.sum"), m.get("dram__bytes_read.sum"), m.get("dram__bytes_write.sum"))
PY
