# smoke, the tests touched since the last full run, the full bench line and the reference arm
mkdir -p gpurun_out
TAG=${TAG:-bf}
timeout 300 python __graft_entry__.py > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log; tail -2 gpurun_out/smoke_$TAG.log
timeout 900 python -m pytest tests/test_torch_ops.py tests/test_gpu_quantile.py -q -x > gpurun_out/pt_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pt_$TAG.log; tail -2 gpurun_out/pt_$TAG.log
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; echo "ref rc=$?"
python - <<PY
import json
d = json.load(open('gpurun_out/bench_$TAG.json'))
print('value', d['value'], 'ms', d['ms_per_step'], 'e2e', d['e2e']['value'], 'frac', d['roofline']['frac'])
for k in ('config3', 'config4b', 'config5'):
    v = d.get(k)
    if isinstance(v, dict): print(k, json.dumps(v)[:400])
r = json.load(open('gpurun_out/bench_ref_$TAG.json')); print('ref', r.get('value'), r.get('unit'))
PY
