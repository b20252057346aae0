#!/usr/bin/env bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_replay.py -q -rfE > gpurun_out/r2e_pytest.txt 2>&1
echo "pytest rc=$?"; tail -5 gpurun_out/r2e_pytest.txt
timeout 1200 python bench.py --steps 10 --warmup 3 --skip-ingest --skip-config4 --skip-config1 --skip-list --skip-config3 --no-cpu > gpurun_out/r2e_bench.json 2> gpurun_out/r2e_bench.err
echo "bench rc=$?"; tail -5 gpurun_out/r2e_bench.err
