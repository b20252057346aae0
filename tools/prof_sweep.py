"""Run the cfg2 sweep + stage step a few times (for ncu captures)."""
import sys, numpy as np, torch
sys.path.insert(0, ".")
import bench
from paper_2406_14424_b200.gridsweep import GridSweep, pareto_counts
from paper_2406_14424_b200.stage import stage_step
_, cert, corr, grids, cost1 = bench.workload(0)
sw = GridSweep(cert, corr, grids, cost1)
for _ in range(3):
    sw.build(); res = sw.evaluate(n_correct=True)
idx = pareto_counts(res.n_correct, res.mean_cost, sw.n_rec)
x = torch.randn((1_000_000, 1000), device="cuda")
for kind in ("margin", "entropy"):
    r = stage_step(x, 0.05, kind=kind)
torch.cuda.synchronize()
print("done", idx.numel())
