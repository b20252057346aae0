# headline sweep line under the three L2 protocols + the phase probe of each variant build
mkdir -p gpurun_out
TAG=${TAG:-f3}
timeout 900 python -m pytest tests/test_gpu_grid.py tests/test_gpu_fullproduct.py -q -x > gpurun_out/pt_$TAG.log 2>&1; echo rc=$? >> gpurun_out/pt_$TAG.log
tail -2 gpurun_out/pt_$TAG.log
for f in paper_2406_14424_b200/libgearserve_b200_phases_*.so; do
  [ -e "$f" ] || continue
  v=$(basename $f .so); v=${v#libgearserve_b200_phases_}
  for m in write none; do
    PHASE_FLUSH=$m GS_LIB_PATH=$PWD/$f timeout 300 python tools/phase_probe.py > gpurun_out/phase_${TAG}_${v}_$m.txt 2>&1
    echo "== $v $m"; grep -h "timeline" gpurun_out/phase_${TAG}_${v}_$m.txt
  done
done
SKIP="--skip-ingest --skip-config4 --skip-config1 --skip-list --skip-config3 --skip-config5 --skip-config4a --skip-stage --no-cpu"
for m in write clean none; do
  timeout 600 python bench.py --steps 20 --warmup 5 $SKIP --flush $m > gpurun_out/bench_${TAG}_$m.json 2> gpurun_out/bench_${TAG}_$m.err
  python -c "
import json; d=json.load(open('gpurun_out/bench_${TAG}_$m.json'))
print('$m step', round(d['ms_per_step']*1e3,2), 'us parity', d.get('parity_spot_check'), {k: round(v*1e3,2) for k,v in d['breakdown_ms'].items() if k!='timing'})
" || tail -5 gpurun_out/bench_${TAG}_$m.err
done
