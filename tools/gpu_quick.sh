set -x
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_grid.py -q -x > gpurun_out/pytest_grid.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_grid.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --skip-stage > gpurun_out/bench.log 2>&1
TAG=prof_r1e KREGEX="grid_hist|slab_first|grid_eval|colscan" SKIP=0 COUNT=5 bash tools/gpu_prof.sh
