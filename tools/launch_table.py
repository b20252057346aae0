"""Aggregate an ncu --csv launch log: per kernel count, mean duration, DRAM bytes."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
h = rows[hi]
ki, mi, vi, ii = h.index('Kernel Name'), h.index('Metric Name'), h.index('Metric Value'), h.index('ID')
per = collections.OrderedDict()
for r in rows[hi + 1:]:
    per.setdefault((r[ii], r[ki]), {})[r[mi]] = float(r[vi].replace(',', ''))
agg = collections.OrderedDict()
for (i, k), m in per.items():
    agg.setdefault(k[:80], []).append(m)
print(f"{'n':>4} {'avg_us':>9} {'dramR_MB':>9} {'dramW_MB':>9}  kernel")
for k, ms in agg.items():
    n = len(ms)
    t = sum(m.get('gpu__time_duration.sum', 0) for m in ms) / n / 1000
    r = sum(m.get('dram__bytes_read.sum', 0) for m in ms) / n / 1e6
    w = sum(m.get('dram__bytes_write.sum', 0) for m in ms) / n / 1e6
    print(f"{n:4d} {t:9.2f} {r:9.2f} {w:9.2f}  {k}")
