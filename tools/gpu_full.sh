# tests + smoke + bench + launch list + ncu --set full of the top kernels (one GPU)
set -x
mkdir -p gpurun_out
TAG=${TAG:-r1}
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"grid_hist|rowscan_first|colscan|grid_eval|stage_step" -s 5 -c 8 -o gpurun_out/full_$TAG python tools/prof_sweep.py > gpurun_out/full_$TAG.log 2>&1
echo done
