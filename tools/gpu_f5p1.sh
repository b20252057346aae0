# ncu capture of config 4a's pass-1 launch on a mid k0 slice (k0 600..611)
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:f5_pass -s 0 -c 1 -o gpurun_out/f5p1 python tools/time_front5.py 100000 12 600 > gpurun_out/f5p1.log 2>&1
python tools/ncu_summary.py gpurun_out/f5p1.ncu-rep f5_pass
