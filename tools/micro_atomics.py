"""Micro-benchmarks: random-scatter atomics vs streaming read on this GPU."""
import sys, torch
sys.path.insert(0, ".")
import bench
from paper_2406_14424_b200.gridsweep import GridSweep

def t(fn, n=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1000

dev = "cuda"
N = 1_000_000
cells = 101 ** 3
F = torch.zeros((cells, 4), device=dev)
idx = torch.randint(0, cells, (N,), device=dev)
vals = torch.ones((N, 4), device=dev)
print("index_add_ 1M rows x 4 f32 (random) us:", t(lambda: F.index_add_(0, idx, vals)))
idx_s = torch.sort(idx).values
print("index_add_ sorted idx us:", t(lambda: F.index_add_(0, idx_s, vals)))
F1 = torch.zeros(cells, device=dev)
print("index_add_ 1M scalar f32 random us:", t(lambda: F1.index_add_(0, idx, vals[:, 0])))
x = torch.randn(N * 4, dtype=torch.float64, device=dev)
print("sum 32MB f64 us:", t(lambda: x.sum()))
print("memset 16.5MB us:", t(lambda: F.zero_()))
_, cert, corr, grids, cost1 = bench.workload(0)
sw = GridSweep(cert, corr, grids, cost1)
g_b = sw.capture(sw.evaluate(), evaluate=False)
print("build graph us:", t(lambda: g_b.replay()))
