mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:head_certainty -s 16 -c 1 -o gpurun_out/head_k512 python tools/head_probe.py > gpurun_out/head_k512.log 2>&1
ncu -i gpurun_out/head_k512.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv, sys
rows = list(csv.reader(sys.stdin)); h = rows[0]
for r in rows[2:3]:
    for k, v in zip(h, r):
        if any(s in k for s in ('sm__pipe_tensor_cycles_active.avg.pct', 'gpu__time_duration.sum', 'dram__bytes_read.sum', 'lts__t_bytes.sum', 'l1tex__m_xbar2l1tex_read_bytes.sum', 'sm__throughput.avg.pct', 'lts__throughput.avg.pct', 'smsp__pcsamp_warps_issue_stalled', 'sm__warps_active.avg.pct', 'smsp__inst_executed.sum')):
            print(k, v)
"
