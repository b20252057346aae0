"""Phase timing of the four-model sweep kernels (GS_PHASE_TIMING build).
Builds libgearserve_b200_phases.so, runs the cfg2 sweep, and prints per
kernel the distribution over CTAs of each phase stamp (globaltimer, us from
the kernel's first CTA start) and of per-CTA phase durations (clock64)."""
import ctypes, os, sys
import numpy as np
sys.path.insert(0, ".")
from paper_2406_14424_b200 import _build
lib_path = _build.build(phase_timing=True)
os.environ["GS_LIB_PATH"] = str(lib_path)
import torch  # noqa: E402
import bench  # noqa: E402
from paper_2406_14424_b200 import _lib  # noqa: E402
from paper_2406_14424_b200.gridsweep import GridSweep  # noqa: E402

K, CTAS, SLOTS = 3, 1024, 8
names = ["g4_sort", "g4_gather", "g4_eval"]
labels = [["start", "grid in", "tables", "loop done", "scanned", "end"],
          ["start", "segments", "plane built", "row walk", "cluster", "end"],
          ["start", "slab in", "cluster", "tables", "edges", "end"]]
_, cert, corr, grids, cost1 = bench.workload(0)
sw = GridSweep(cert, corr, grids, cost1, build=False)
out = None
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
flush_read = torch.empty(512 << 20, dtype=torch.uint8, device="cuda").fill_(1)
mode = os.environ.get("PHASE_FLUSH", "write")  # write | clean | none
print(f"# flush before each build: {mode}")
for _ in range(5):
    if mode != "none":
        flush.zero_()
    if mode == "clean":
        flush_read.sum()
    sw.build()
    out = sw.evaluate(out=out)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (K * CTAS * SLOTS * 2))()
assert _lib.load().gs_debug_phases(buf) == 0
a = np.frombuffer(buf, dtype=np.uint64).reshape(K, CTAS, SLOTS, 2).astype(np.float64)
clk = float(os.environ.get("SM_MHZ", "1965"))
for k in range(K):
    g, c = a[k, :, :, 0], a[k, :, :, 1]
    live = g[:, 0] > 0
    g, c = g[live], c[live]
    t0 = g[:, 0].min()
    print(f"== {names[k]}: {live.sum()} CTAs, kernel span {(g.max() - t0) / 1e3:.2f} us")
    for s, lab in enumerate(labels[k]):
        col = g[:, s]
        ok = col > 0
        if not ok.any():
            continue
        rel = (col[ok] - t0) / 1e3
        dur = (c[ok, s] - c[ok, 0]) / clk
        print(f"   {s} {lab:10s} t[us] min {rel.min():6.2f} med {np.median(rel):6.2f} max {rel.max():6.2f}"
              f" | since start[us] med {np.median(dur):6.2f} max {dur.max():6.2f}")
