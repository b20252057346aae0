mkdir -p gpurun_out
timeout 300 python tools/time_front5.py 100000 40 2>&1 | tail -3
timeout 900 ncu --set full --clock-control none --import-source on -k regex:f5_pass -c 1 -o gpurun_out/f5pass python tools/time_front5.py 100000 8 > gpurun_out/f5pass_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/f5pass.ncu-rep f5_pass
python tools/sass_windows.py gpurun_out/f5pass.ncu-rep f5_pass 0x100 2>&1 | sort -t'%' -k3 -rn | head -30
