"""Run the cfg2 sweep + stage step a few times (for ncu captures)."""
import sys, numpy as np, torch
sys.path.insert(0, ".")
import bench
from paper_2406_14424_b200.gridsweep import GridSweep, pareto_counts
_, cert, corr, grids, cost1 = bench.workload(0)
sw = GridSweep(cert, corr, grids, cost1)
for _ in range(3):
    sw.build(); res = sw.evaluate(n_correct=True)
for _ in range(2):
    idx = pareto_counts(res.n_correct, res.mean_cost, sw.n_rec)
torch.cuda.synchronize()
print("done", idx.numel())
