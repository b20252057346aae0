"""Step time of the cfg2 sweep (one graph: flush, event, sweep, event) with
torch's fill as the flush vs gs_flush_l2 (default / max carveout)."""
import sys
import torch
sys.path.insert(0, ".")
import bench
from paper_2406_14424_b200 import _lib
from paper_2406_14424_b200.gridsweep import GridSweep

_, cert, corr, grids, cost1 = bench.workload(0)
sw = GridSweep(cert, corr, grids, cost1)
out = sw.evaluate()
buf = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
lib = _lib.load()
x = torch.zeros(1, device="cuda")
for name, fl in [("torch fill", lambda: buf.zero_()),
                 ("gs_flush default", lambda: lib.gs_flush_l2(buf.data_ptr(), buf.numel(), 0, _lib.stream_ptr())),
                 ("gs_flush max carveout", lambda: lib.gs_flush_l2(buf.data_ptr(), buf.numel(), 1, _lib.stream_ptr()))]:
    for body_name, body in [("sweep", lambda: (sw.build(), sw.evaluate(out=out))), ("trivial", lambda: x.add_(1))]:
        ev = (torch.cuda.Event(enable_timing=True, external=True), torch.cuda.Event(enable_timing=True, external=True))
        fl(); body(); torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fl()
            ev[0].record()
            body()
            ev[1].record()
        ts = []
        for i in range(25):
            g.replay()
            torch.cuda.synchronize()
            if i >= 5:
                ts.append(ev[0].elapsed_time(ev[1]) * 1e3)
        ts.sort()
        print(f"{name:22s} {body_name:8s} median {ts[len(ts)//2]:7.2f} us  best {ts[0]:7.2f} us")
