mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:engine_kernel -s 1 -c 1 -o gpurun_out/engine python tools/prof_engine.py > gpurun_out/engine_ncu.log 2>&1
python tools/ncu_summary.py gpurun_out/engine.ncu-rep engine
python tools/sass_windows.py gpurun_out/engine.ncu-rep engine 0x200 2>&1 | head -40
