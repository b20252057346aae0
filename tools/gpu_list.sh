mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_eval.py tests/test_gpu_cascades.py -q -x > gpurun_out/pt_list.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pt_list.log; tail -2 gpurun_out/pt_list.log
timeout 900 python bench.py --steps 3 --warmup 3 --skip-ingest --skip-config4 --skip-config1 --skip-config3 --skip-config5 --skip-config4a --skip-stage --skip-head --no-cpu > gpurun_out/bench_list.json 2> gpurun_out/bench_list.err
python -c "
import json; d=json.load(open('gpurun_out/bench_list.json')); l=d['list_path']; print('pub', l['published_point']['device_ms'], l['published_point']['e2e_ms_median']); print('sp1', json.dumps(l['sp1_shape'])[:600])" || tail -3 gpurun_out/bench_list.err
