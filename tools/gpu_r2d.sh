#!/usr/bin/env bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_sampler.py tests/test_gpu_reference_suite.py -q -rfE > gpurun_out/r2d_pytest.txt 2>&1
echo "pytest rc=$?"; tail -30 gpurun_out/r2d_pytest.txt
