#!/usr/bin/env bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_grid.py tests/test_gpu_replay.py -q -x -rfE -k "five or config4b or random_grids or ranges or 65535 or replay or scenario or launch or metrics" > gpurun_out/r2f_pytest.txt 2>&1
echo "pytest rc=$?"; tail -5 gpurun_out/r2f_pytest.txt
bash tools/gpu_w5prof.sh 2>&1 | grep -v "^$" | tail -8
timeout 900 python - <<'PY' > gpurun_out/r2f_bench.txt 2>&1
import sys, json, argparse
sys.path.insert(0, ".")
import bench, torch
args = argparse.Namespace(steps=5, warmup=3)
d = bench.config4_bench(args, torch.device("cuda", 0))
print("cfg4b", d["ms"], d["frac"], d["parity_spot_check"])
d = bench.config5_bench(args, torch.device("cuda", 0))
print("cfg5", d["ms"], d["routed_samples_per_s"], d["parity_prefix"], d["probes"]["ms"], d["probes"]["probes_per_s"])
PY
cat gpurun_out/r2f_bench.txt | tail -3
