mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_front5.py -q -x > gpurun_out/pt_f5.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pt_f5.log; tail -2 gpurun_out/pt_f5.log
timeout 300 python tools/time_front5.py 100000 40 2>&1 | tail -3
timeout 900 python bench.py --steps 3 --warmup 3 --skip-ingest --skip-config4 --skip-config1 --skip-list --skip-config3 --skip-config5 --skip-stage --skip-head --no-cpu > gpurun_out/bench_f5.json 2> gpurun_out/bench_f5.err
python -c "
import json; d=json.load(open('gpurun_out/bench_f5.json')); c=d['config4a']; print({k: c.get(k) for k in ('seconds','config_evals_per_s','front_points','front_configs','spot_check_vs_oracle')})" || tail -3 gpurun_out/bench_f5.err
