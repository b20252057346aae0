mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stage.py tests/test_gpu_cascades.py tests/test_gpu_eval.py -q -x > gpurun_out/pt_st2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pt_st2.log; tail -2 gpurun_out/pt_st2.log
timeout 900 python bench.py --steps 3 --warmup 3 --skip-ingest --skip-config4 --skip-config1 --skip-list --skip-config5 --skip-config4a --skip-head --no-cpu > gpurun_out/bench_st2.json 2> gpurun_out/bench_st2.err
python -c "
import json; d=json.load(open('gpurun_out/bench_st2.json')); print(json.dumps(d.get('stage_step')))" || tail -3 gpurun_out/bench_st2.err
