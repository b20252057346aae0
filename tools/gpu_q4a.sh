mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_quantile.py tests/test_torch_ops.py -q -x > gpurun_out/pt_q4a.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pt_q4a.log; tail -3 gpurun_out/pt_q4a.log
timeout 900 python bench.py --steps 3 --warmup 3 --skip-ingest --skip-config4 --skip-config1 --skip-list --skip-config3 --skip-config5 --skip-stage --skip-head --no-cpu > gpurun_out/bench_q4a.json 2> gpurun_out/bench_q4a.err
python -c "
import json; d=json.load(open('gpurun_out/bench_q4a.json')); print(json.dumps(d.get('config4a'))[:1500])"
