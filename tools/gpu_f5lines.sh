mkdir -p gpurun_out
timeout 300 python tools/time_front5.py 100000 12 600 2>&1 | grep "k0 \["
timeout 900 ncu --set full --clock-control none --import-source on -k regex:f5_pass -s 1 -c 1 -o gpurun_out/f5mid python tools/time_front5.py 100000 12 600 > gpurun_out/f5mid.log 2>&1
python tools/ncu_summary.py gpurun_out/f5mid.ncu-rep f5_pass
python tools/sass_lines.py gpurun_out/f5mid.ncu-rep f5_pass paper_2406_14424_b200/_objs/gs_front5.o 25
