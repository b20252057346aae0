set -x
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_stage.py tests/test_gpu_engine.py -q -x > gpurun_out/pytest_stage.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_stage.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"stage_step" -s 2 -c 2 -o gpurun_out/prof_stage python tools/prof_sweep.py > gpurun_out/prof_stage.log 2>&1
