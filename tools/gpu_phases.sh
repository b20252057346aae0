# phase probe of every variant build (2 runs each), no tests
mkdir -p gpurun_out
for f in paper_2406_14424_b200/libgearserve_b200_phases_*.so; do
  v=$(basename $f .so); v=${v#libgearserve_b200_phases_}
  for rep in 1 2; do
    GS_LIB_PATH=$PWD/$f timeout 300 python tools/phase_probe.py > gpurun_out/phase_v_${v}_$rep.txt 2>&1
    echo "== $v run $rep"; grep -h "timeline g4_eval" gpurun_out/phase_v_${v}_$rep.txt
  done
done
