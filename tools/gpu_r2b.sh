#!/usr/bin/env bash
mkdir -p gpurun_out
free -g > gpurun_out/r2b_free.txt
timeout 900 python -m pytest tests/test_gpu_fullproduct.py tests/test_gpu_stage.py -q -rfE > gpurun_out/r2b_pytest.txt 2>&1
echo "pytest rc=$?"; tail -5 gpurun_out/r2b_pytest.txt
timeout 1200 python bench.py --steps 20 --warmup 5 --skip-ingest --skip-config4 > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err
echo "bench rc=$?"; tail -20 gpurun_out/r2b_bench.err
