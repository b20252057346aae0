mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_stage.py -q -x > gpurun_out/pt_router.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pt_router.log; tail -2 gpurun_out/pt_router.log
timeout 900 python -m pytest tests/test_gpu_reference_suite.py -q -x -k "engine" > gpurun_out/pt_router_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/pt_router_ref.log; tail -2 gpurun_out/pt_router_ref.log
timeout 600 python tools/router_probe.py 2>&1 | grep "per call"
timeout 900 python bench.py --steps 3 --warmup 3 --skip-ingest --skip-config4 --skip-config1 --skip-list --skip-config3 --skip-config4a --skip-stage --skip-head --no-cpu > gpurun_out/bench_router.json 2> gpurun_out/bench_router.err
python -c "
import json; d=json.load(open('gpurun_out/bench_router.json')); print(json.dumps(d['config5'].get('online_router'))[:900])" || tail -3 gpurun_out/bench_router.err
