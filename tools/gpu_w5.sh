#!/usr/bin/env bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_grid.py -q -x -rfE > gpurun_out/w5_pytest.txt 2>&1
echo "pytest rc=$?"; tail -15 gpurun_out/w5_pytest.txt
timeout 900 python - <<'PY' > gpurun_out/w5_bench.txt 2>&1
import sys, json, argparse
sys.path.insert(0, ".")
import bench, torch
args = argparse.Namespace(steps=5, warmup=3)
print(json.dumps(bench.config4_bench(args, torch.device("cuda", 0)), indent=1))
PY
cat gpurun_out/w5_bench.txt | tail -30
