"""Fixed overhead of a timed step: event->event time of the cfg2 sweep step
as one CUDA graph vs direct stream launches, and of a trivial graph, each
after the 512 MB write flush (bench.py's timing, without the clocks)."""
import sys
import torch
sys.path.insert(0, ".")
import bench
from paper_2406_14424_b200.gridsweep import GridSweep

_, cert, corr, grids, cost1 = bench.workload(0)
sw = GridSweep(cert, corr, grids, cost1)
out = sw.evaluate()
g_step = sw.capture(out)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
x = torch.zeros(1, device="cuda")
g_triv = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    x.add_(1)
torch.cuda.current_stream().wait_stream(s)
with torch.cuda.graph(g_triv):
    x.add_(1)


def timed(fn, n=20, warm=5):
    st = torch.cuda.current_stream()
    res = []
    for i in range(n + warm):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        fn()
        b.record(st)
        torch.cuda.synchronize()
        if i >= warm:
            res.append(a.elapsed_time(b) * 1e3)
    res.sort()
    return res[len(res) // 2], res[0]


for name, fn in [("step graph", g_step.replay), ("step direct", lambda: (sw.build(), sw.evaluate(out=out))),
                 ("trivial graph", g_triv.replay), ("trivial kernel", lambda: x.add_(1)),
                 ("build graph-less", sw.build), ("eval graph-less", lambda: sw.evaluate(out=out))]:
    med, best = timed(fn)
    print(f"{name:18s} median {med:7.2f} us  best {best:7.2f} us")
