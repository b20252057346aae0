#!/usr/bin/env bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_front5.py -q -x -rfE 2>&1 | tail -2
timeout 900 python - <<'PY' > gpurun_out/r2h_4a.txt 2>&1
import sys, json, argparse
sys.path.insert(0, ".")
import bench, torch
args = argparse.Namespace(steps=5, warmup=3)
print(json.dumps(bench.config4a_bench(args, torch.device("cuda", 0), 1, 0), indent=1))
PY
tail -30 gpurun_out/r2h_4a.txt
