mkdir -p gpurun_out
TAG=${TAG:-q}
timeout 900 python -m pytest tests/test_gpu_quantile.py tests/test_gpu_cascades.py -q -x > gpurun_out/pt_$TAG.log 2>&1; echo rc=$? >> gpurun_out/pt_$TAG.log
tail -3 gpurun_out/pt_$TAG.log
timeout 300 python tools/quantile_probe.py > gpurun_out/qprobe_$TAG.txt 2>&1; cat gpurun_out/qprobe_$TAG.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"select|gather_pass0|pass1|resolve|plan_rows|collect|lerp|init_targets" --csv --log-file gpurun_out/qlaunch_$TAG.csv python tools/quantile_probe.py > /dev/null 2>&1
python - <<PY
import csv, collections
rows = list(csv.reader(open('gpurun_out/qlaunch_$TAG.csv')))
i = next(i for i, r in enumerate(rows) if 'Kernel Name' in r); h = rows[i]; c = {k: j for j, k in enumerate(h)}
agg = collections.defaultdict(list)
for r in rows[i + 1:]:
    if len(r) == len(h) and r[c['Metric Name']] == 'gpu__time_duration.sum':
        agg[r[c['Kernel Name']][:60]].append(float(r[c['Metric Value']].replace(',', '')))
for k, v in agg.items(): print(f"{k:60s} n={len(v)} mean_us={sum(v)/len(v)/1e3:.2f}")
PY
