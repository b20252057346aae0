#!/usr/bin/env bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_replay.py tests/test_gpu_reference_suite.py tests/test_gpu_engine.py -q -rfE -v > gpurun_out/r2c_pytest.txt 2>&1
echo "pytest rc=$?"; grep -E "PASS|FAIL|ERROR|passed|failed" gpurun_out/r2c_pytest.txt | tail -30
