#!/usr/bin/env bash
# phase probes of the variant libraries + a headline bench line
mkdir -p gpurun_out
for f in paper_2406_14424_b200/libgearserve_b200_phases_*.so; do
  tag=$(basename $f .so); tag=${tag#libgearserve_b200_phases_}
  for rep in 1 2; do
    GS_LIB_PATH=$PWD/$f timeout 300 python tools/phase_probe.py > gpurun_out/exp_${tag}_${rep}.txt 2>&1
  done
  echo "== $tag"; grep -h "timeline" gpurun_out/exp_${tag}_*.txt
done
if [ -z "$NO_BENCH" ]; then
timeout 600 python bench.py --steps 20 --warmup 5 --skip-ingest --skip-config4 --skip-config1 --skip-list --skip-config3 --skip-config5 --no-cpu > gpurun_out/exp_bench.json 2> gpurun_out/exp_bench.err
python -c "
import json; d=json.load(open('gpurun_out/exp_bench.json'))
print('step', d['ms_per_step'], 'stream', d['ms_per_step_stream_events'], 'value', d['value'], 'parity', d['parity_spot_check'], d['breakdown_ms'])
"
fi
