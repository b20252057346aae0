"""Config-4b build and eval times (5 models, 100-level grids, 100k records),
CUDA events, median of 10: python tools/w5_probe.py"""
import sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_2406_14424_b200 import synth
from paper_2406_14424_b200.cascades import grid_values
from paper_2406_14424_b200.gridsweep import GridSweep
cert, corr = synth.validation_matrices(5, 100_000, 0.8, 5)
grids = [np.array(grid_values(cert[:, j], 100)) for j in range(5)]
sw = GridSweep(cert, corr, grids, np.array([1.0, 4.0, 16.0, 64.0, 256.0]))
out = sw.evaluate()
ref = out.accuracy.clone()
ts, te = [], []
for i in range(12):
    a, b, c = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    a.record(); sw.build(); b.record(); sw.evaluate(out=out); c.record()
    torch.cuda.synchronize()
    if i >= 2: ts.append(a.elapsed_time(b)); te.append(b.elapsed_time(c))
print(f"build {np.median(ts)*1e3:.0f} us eval {np.median(te)*1e3:.0f} us same={torch.equal(out.accuracy, ref)}")
