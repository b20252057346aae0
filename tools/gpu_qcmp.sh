mkdir -p gpurun_out
echo "== radix select (this build)"; timeout 300 python tools/quantile_probe.py
echo "== CUB sort (previous build)"; GS_LIB_PATH=$PWD/paper_2406_14424_b200/libgearserve_b200_oldq.so timeout 300 python tools/quantile_probe.py
