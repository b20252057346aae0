#!/usr/bin/env bash
# round-2 check: full GPU test suite (incl. the reference suite through the
# binding and the full-product proof), sanitizers, one bench line.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2_smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rfE --durations=20 > gpurun_out/r2_pytest.txt 2>&1
echo "pytest rc=$?"
tail -30 gpurun_out/r2_pytest.txt
bash tools/gpu_sanitize.sh > gpurun_out/r2_sanitize.txt 2>&1
cat gpurun_out/r2_sanitize.txt
timeout 900 python bench.py --steps 20 --warmup 5 --skip-ingest > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err
echo "bench rc=$?"
head -c 1500 gpurun_out/r2_bench.json
