# ncu --set full capture of the sweep + stage-step kernels (one GPU)
set -x
mkdir -p gpurun_out
TAG=${TAG:-prof}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-grid_hist|slab_scan|scan_dim|grid_eval|stage_step}" -s ${SKIP:-4} -c ${COUNT:-8} -o gpurun_out/$TAG python tools/prof_sweep.py > gpurun_out/$TAG.log 2>&1
echo "rc=$?"
