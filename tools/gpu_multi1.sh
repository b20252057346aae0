#!/usr/bin/env bash
# the torchrun (N = 2) bench path on one GPU: gloo, both ranks on cuda:0
mkdir -p gpurun_out
GS_ONE_DEVICE=1 GS_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu \
  --skip-ingest --skip-config4 --skip-config1 --skip-list --skip-config3 --skip-config5 \
  > gpurun_out/multi1.json 2> gpurun_out/multi1.err
echo "rc=$?"; tail -5 gpurun_out/multi1.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/multi1.json").read().strip().splitlines()[-1])
print("n_gpus", d["n_gpus"], "value", d["value"], "step", d["ms_per_step"], "e2e", d["e2e"]["value"])
print(json.dumps(d.get("config4a"))[:600])
PY
