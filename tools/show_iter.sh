TAG=${TAG:-s1}
tail -1 gpurun_out/pt_$TAG.log
for f in write clean; do tail -1 gpurun_out/bench_${TAG}_$f.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('$f', round(d['ms_per_step']*1e3,2), 'us', round(d['value']/1e9,2), 'G/s frac', round(d['roofline']['step']['frac'],3))"; done
head -${N:-20} gpurun_out/phase_$TAG.txt
