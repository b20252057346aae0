#!/usr/bin/env bash
# full GPU suite + full bench line
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -rfE --durations=15 > gpurun_out/r2g_pytest.txt 2>&1
echo "pytest rc=$?"; tail -25 gpurun_out/r2g_pytest.txt
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/r2g_bench.json 2> gpurun_out/r2g_bench.err
echo "bench rc=$?"; tail -5 gpurun_out/r2g_bench.err
python - <<'PY'
import json
d = json.load(open("gpurun_out/r2g_bench.json"))
print("step", d["ms_per_step"], "value", d["value"], "frac", d["roofline"]["frac"], "parity", d["parity_spot_check"])
for k in ("config1", "config3", "config4b", "config5", "list_path", "ingest", "stage_step"):
    v = d.get(k)
    print(k, json.dumps(v)[:300] if v else None)
PY
