mkdir -p gpurun_out
TAG=${TAG:-tc}
timeout 600 python -m pytest tests/test_gpu_head.py -q -x > gpurun_out/pt_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pt_$TAG.log
tail -30 gpurun_out/pt_$TAG.log
timeout 300 python tools/head_probe.py 2>&1 | tail -8
