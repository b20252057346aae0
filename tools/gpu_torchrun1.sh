mkdir -p gpurun_out
GS_ONE_DEVICE=1 GS_DIST_BACKEND=gloo timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --steps 5 --warmup 3 --skip-ingest --skip-config1 --skip-list --skip-config3 --skip-config5 --skip-stage --no-cpu > gpurun_out/torchrun2.json 2> gpurun_out/torchrun2.err; echo "rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/torchrun2.json')); print('n_gpus', d['n_gpus'], 'value', d['value'], 'scaling', d['scaling']); print(json.dumps(d.get('config4a'))[:600]); print(json.dumps(d.get('head'))[:300])" || tail -20 gpurun_out/torchrun2.err
