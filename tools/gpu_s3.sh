# session-3 iteration on one GPU: four-model parity tests, phase probes of the
# variant builds (tools/exp_variants.sh), the headline sweep line
mkdir -p gpurun_out
TAG=${TAG:-s3}
timeout 900 python -m pytest tests/test_gpu_grid.py tests/test_gpu_fullproduct.py -q -x ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pt_$TAG.log 2>&1; echo rc=$? >> gpurun_out/pt_$TAG.log
tail -3 gpurun_out/pt_$TAG.log
for f in paper_2406_14424_b200/libgearserve_b200_phases_*.so; do
  [ -e "$f" ] || continue
  v=$(basename $f .so); v=${v#libgearserve_b200_phases_}
  GS_LIB_PATH=$PWD/$f timeout 300 python tools/phase_probe.py > gpurun_out/phase_${TAG}_$v.txt 2>&1
  echo "== $v"; grep -h "timeline" gpurun_out/phase_${TAG}_$v.txt
done
timeout 600 python bench.py --steps 20 --warmup 5 --skip-ingest --skip-config4 --skip-config1 --skip-list --skip-config3 --skip-config5 --skip-config4a --skip-stage --no-cpu > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
python -c "
import json; d=json.load(open('gpurun_out/bench_$TAG.json'))
print('step', d['ms_per_step'], 'stream', d['ms_per_step_stream_events'], 'value', d['value'], 'parity', d['parity_spot_check'], d['breakdown_ms'])
" || tail -5 gpurun_out/bench_$TAG.err
