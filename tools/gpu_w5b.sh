#!/usr/bin/env bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_grid.py -q -x -rfE -k "five or config4b or random_grids or ranges or 65535" > gpurun_out/w5_pytest.txt 2>&1
echo "pytest rc=$?"; tail -5 gpurun_out/w5_pytest.txt
bash tools/gpu_w5prof.sh 2>&1 | grep -v "^$" | tail -8
timeout 900 python - <<'PY' > gpurun_out/w5_bench.txt 2>&1
import sys, json, argparse
sys.path.insert(0, ".")
import bench, torch
args = argparse.Namespace(steps=5, warmup=3)
d = bench.config4_bench(args, torch.device("cuda", 0))
print(d["ms"], d["frac"], d["parity_spot_check"])
PY
cat gpurun_out/w5_bench.txt | tail -3
