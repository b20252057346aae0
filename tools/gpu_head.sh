# quick state check of HEAD on one GPU: smoke, the GPU suite, the headline sweep line
mkdir -p gpurun_out
TAG=${TAG:-h}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/nvsmi_$TAG.txt
timeout 300 python __graft_entry__.py > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
tail -2 gpurun_out/smoke_$TAG.log
timeout 1200 python -m pytest tests -q -m gpu --durations=15 > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
tail -4 gpurun_out/pytest_gpu_$TAG.log
timeout 600 python bench.py --steps 20 --warmup 5 --skip-ingest --skip-config4 --skip-config1 --skip-list --skip-config3 --skip-config5 --skip-config4a --skip-stage --no-cpu > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
python -c "
import json; d=json.load(open('gpurun_out/bench_$TAG.json'))
print('step', d['ms_per_step'], 'value', d['value'], 'parity', d.get('parity_spot_check'), d.get('breakdown_ms'))
" || tail -5 gpurun_out/bench_$TAG.err
timeout 300 python tools/phase_probe.py > gpurun_out/phase_$TAG.txt 2>&1; grep -h timeline gpurun_out/phase_$TAG.txt
