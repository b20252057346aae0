#!/usr/bin/env bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_grid.py tests/test_gpu_fullproduct.py -q -x > gpurun_out/exp2_pytest.txt 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/exp2_pytest.txt
NO_BENCH=1 bash tools/gpu_exp.sh
for f in gpurun_out/exp_lut_1.txt; do sed -n 1,12p $f; done
timeout 600 python bench.py --steps 20 --warmup 5 --skip-ingest --skip-config4 --skip-config1 --skip-list --skip-config3 --skip-config5 --no-cpu > gpurun_out/exp_bench.json 2> gpurun_out/exp_bench.err
python -c "
import json; d=json.load(open('gpurun_out/exp_bench.json'))
print('step', d['ms_per_step'], 'stream', d['ms_per_step_stream_events'], 'value', d['value'], 'parity', d['parity_spot_check'], d['breakdown_ms'])
"
