"""e2e variants of the cfg2 sweep from pinned host matrices (timing probe)."""
import sys, time
import numpy as np, torch
sys.path.insert(0, ".")
import bench
from paper_2406_14424_b200.gridsweep import GridSweep, front_host, pareto_counts

_, cert, corr, grids, cost1 = bench.workload(0)
pc = torch.from_numpy(cert).pin_memory()
pk = torch.from_numpy(corr).pin_memory()
dc = torch.empty_like(pc, device="cuda")
dk = torch.empty_like(pk, device="cuda")
sw = GridSweep(dc, dk, grids, cost1, build=False)
out = None


def plain():
    dc.copy_(pc, non_blocking=True)
    dk.copy_(pk, non_blocking=True)
    sw.build()


def streamed(k):
    return lambda: sw.build_streamed(pc, pk, chunks=k)


def step(build):
    global out
    build()
    out = sw.evaluate(n_correct=True, out=out)
    idx = pareto_counts(out.n_correct, out.mean_cost, sw.n_rec)
    return front_host(idx, out)


def timeit(f, n=20):
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        f()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / n


print("copy only      %.3f ms" % timeit(lambda: (dc.copy_(pc, non_blocking=True), dk.copy_(pk, non_blocking=True))))
print("plain build    %.3f ms" % timeit(plain))
for k in (2, 4, 8, 16):
    print("streamed %2d    %.3f ms" % (k, timeit(streamed(k))))
print("e2e plain      %.3f ms" % timeit(lambda: step(plain)))
for k in (4, 8):
    print("e2e streamed %d %.3f ms" % (k, timeit(lambda: step(streamed(k)))))
print("eval+pareto+d2h %.3f ms" % timeit(lambda: step(lambda: None)))
plain()
out = sw.evaluate(n_correct=True, out=out)
print("eval only       %.3f ms" % timeit(lambda: sw.evaluate(n_correct=True, out=out)))
print("pareto (+sync)  %.3f ms" % timeit(lambda: pareto_counts(out.n_correct, out.mean_cost, sw.n_rec)))
idx = pareto_counts(out.n_correct, out.mean_cost, sw.n_rec)
print("front rows+D2H  %.3f ms (n_front %d)" % (timeit(lambda: front_host(idx, out)), idx.numel()))
