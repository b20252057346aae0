# quick iteration on one GPU: grid parity tests, bench (both flushes, sweep only), phase probe
mkdir -p gpurun_out
TAG=${TAG:-s1}
timeout 600 python -m pytest tests/test_gpu_grid.py tests/test_gpu_cascades.py -q -x > gpurun_out/pt_$TAG.log 2>&1; echo rc=$? >> gpurun_out/pt_$TAG.log
for f in write clean; do
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --skip-stage --skip-ingest --skip-config4 --skip-config1 --flush $f > gpurun_out/bench_${TAG}_$f.log 2>&1
done
timeout 300 python tools/phase_probe.py > gpurun_out/phase_$TAG.txt 2>&1
if [ -n "$AB" ]; then env $AB timeout 300 python tools/phase_probe.py > gpurun_out/phase_${TAG}_ab.txt 2>&1; env $AB timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --skip-stage --skip-ingest --skip-config4 --skip-config1 > gpurun_out/bench_${TAG}_ab.log 2>&1; fi
tail -2 gpurun_out/pt_$TAG.log
