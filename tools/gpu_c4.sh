# five-model path: parity tests (incl. the full 4b product vs the general path) and the config-4b bench leg
mkdir -p gpurun_out
TAG=${TAG:-c4}
timeout 900 python -m pytest tests/test_gpu_grid.py -q -x -k "five or 4b" > gpurun_out/pt_$TAG.log 2>&1; echo rc=$? >> gpurun_out/pt_$TAG.log
tail -3 gpurun_out/pt_$TAG.log
timeout 600 python bench.py --steps 5 --warmup 3 --skip-ingest --skip-config1 --skip-list --skip-config3 --skip-config5 --skip-config4a --skip-stage --no-cpu > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
python -c "
import json; d=json.load(open('gpurun_out/bench_$TAG.json')); c=d['config4b']
print('cfg4b ms', c['ms'], 'frac', c['frac'], 'parity', c['parity_spot_check'])
" || tail -5 gpurun_out/bench_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"w5_|grid_eval" --csv --log-file gpurun_out/launches_$TAG.csv python tools/prof_cfg4.py > /dev/null 2>&1
python - <<PY
import csv, collections
rows = list(csv.reader(open('gpurun_out/launches_$TAG.csv')))
i = next(i for i, r in enumerate(rows) if 'Kernel Name' in r); h = rows[i]; c = {k: j for j, k in enumerate(h)}
agg = collections.defaultdict(list)
for r in rows[i + 1:]:
    if len(r) == len(h) and r[c['Metric Name']] == 'gpu__time_duration.sum':
        agg[r[c['Kernel Name']][:50]].append(float(r[c['Metric Value']].replace(',', '')))
for k, v in agg.items(): print(f"{k:50s} n={len(v)} mean_us={sum(v)/len(v)/1e3:.1f}")
PY
