mkdir -p gpurun_out
python tools/list_probe.py
timeout 600 ncu --set full --clock-control none --import-source on -k regex:eval_list -s 2 -c 1 -o gpurun_out/listsp1 python tools/list_probe.py > gpurun_out/listsp1.log 2>&1
python tools/ncu_summary.py gpurun_out/listsp1.ncu-rep eval_list
