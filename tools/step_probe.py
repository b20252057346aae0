"""Config-2 headline step (build + eval; 512 MB write flush before each
step; events inside one graph, as bench.py), median over 100 steps, for
same-box A/B of library builds: GS_LIB_PATH=... python tools/step_probe.py"""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2406_14424_b200.gridsweep import GridSweep  # noqa: E402

_, cert, corr, grids, cost1 = bench.workload(seed=0)
sw = GridSweep(cert, corr, grids, cost1)
out = sw.evaluate()
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
ev = (torch.cuda.Event(enable_timing=True, external=True), torch.cuda.Event(enable_timing=True, external=True))
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    flush.zero_()
    ev[0].record()
    sw.build()
    sw.evaluate(out=out)
    ev[1].record()
for _ in range(10):
    g.replay()
torch.cuda.synchronize()
ts = []
for _ in range(100):
    g.replay()
    torch.cuda.synchronize()
    ts.append(ev[0].elapsed_time(ev[1]) * 1e3)
print(f"step us: median {np.median(ts):.2f} mean {np.mean(ts):.2f} min {np.min(ts):.2f}")
