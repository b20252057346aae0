mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_eval.py tests/test_gpu_cascades.py tests/test_gpu_reference_suite.py -q -x 2>&1 | tail -2
timeout 600 python bench.py --steps 3 --warmup 3 --skip-ingest --skip-config4 --skip-config4a --skip-config1 --skip-config3 --skip-config5 --skip-stage --skip-head --no-cpu > gpurun_out/bench_list2.json 2> gpurun_out/bench_list2.err
python -c "
import json; d=json.load(open('gpurun_out/bench_list2.json')); l=d['list_path']; print(l['published_point'].get('device_ms'), l['published_point'].get('bit_exact_vs_oracle'), l['sp1_shape'].get('device_ms'), l['sp1_shape'].get('parity_spot_check'))" || tail -3 gpurun_out/bench_list2.err
