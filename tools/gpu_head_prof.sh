mkdir -p gpurun_out
TAG=${TAG:-hp}
timeout 900 python bench.py --steps 5 --warmup 3 --skip-ingest --skip-config4 --skip-config1 --skip-list --skip-config3 --skip-config5 --skip-config4a --skip-stage --no-cpu > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
python -c "
import json; d=json.load(open('gpurun_out/bench_$TAG.json')); print(json.dumps(d.get('head'), indent=1))" || tail -5 gpurun_out/bench_$TAG.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:head_certainty -s 3 -c 1 -o gpurun_out/head_$TAG python tools/head_probe.py > gpurun_out/head_ncu_$TAG.log 2>&1
ncu -i gpurun_out/head_$TAG.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv, sys
rows = list(csv.reader(sys.stdin)); h = rows[0]
for r in rows[2:3]:
    for k, v in zip(h, r):
        if any(s in k for s in ('pipe_tensor', 'gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'sm__throughput.avg.pct', 'launch__grid_size', 'launch__registers', 'sm__inst_executed_pipe_uniform', 'lts__t_bytes.sum')):
            print(k, v)
" > gpurun_out/head_metrics_$TAG.txt; cat gpurun_out/head_metrics_$TAG.txt
