#!/usr/bin/env bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_front5.py -q -x -rfE > gpurun_out/f5_pytest.txt 2>&1
echo "pytest rc=$?"; tail -15 gpurun_out/f5_pytest.txt
timeout 600 python tools/time_front5.py 100000 100 2>&1 | tail -4
