#!/usr/bin/env bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stage.py -q -x -rfE -k config3_scale 2>&1 | tail -3
timeout 900 python - <<'PY' > gpurun_out/r2i_cfg5.txt 2>&1
import sys, json, argparse
sys.path.insert(0, ".")
import bench, torch
args = argparse.Namespace(steps=5, warmup=3)
d = bench.config5_bench(args, torch.device("cuda", 0))
print(json.dumps(d["online_router"], indent=1))
print(d["ms"], d["routed_samples_per_s"], d["probes"]["ms"])
PY
tail -40 gpurun_out/r2i_cfg5.txt
