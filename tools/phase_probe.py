"""Phase timing of the four-model sweep kernels (GS_PHASE_TIMING build).
Builds libgearserve_b200_phases.so, runs the cfg2 sweep, and prints per
kernel the distribution over CTAs of each phase stamp (globaltimer, us from
the kernel's first CTA start) and of per-CTA phase durations (clock64)."""
import ctypes, os, sys
import numpy as np
sys.path.insert(0, ".")
from paper_2406_14424_b200 import _build
if not os.environ.get("GS_LIB_PATH"):
    os.environ["GS_LIB_PATH"] = str(_build.build(phase_timing=True))
import torch  # noqa: E402
import bench  # noqa: E402
from paper_2406_14424_b200 import _lib  # noqa: E402
from paper_2406_14424_b200.gridsweep import GridSweep  # noqa: E402

K, CTAS, SLOTS = 3, 1024, 8
names = ["g4_sort", "g4_gather", "g4_eval"]
labels = [["start", "grid in", "tables", "loop done", "scanned", "end"],
          ["start", "segments", "plane built", "row walk", "cluster", "end"],
          ["start", "staged", "unit 1", "unit 2", "unit 3", "end"]]
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
# timeline of the last build + eval: each kernel's first CTA start and last
# stamp, from the first kernel's first start (the stamps are overwritten by
# every launch, so these are the last iteration's)
T0 = min(a[k, :, 0, 0][a[k, :, 0, 0] > 0].min() for k in range(K))
for k in range(K):
    g = a[k, :, :, 0]
    live = g[:, 0] > 0
    print(f"# timeline {names[k]:10s} first start {(g[live, 0].min() - T0) / 1e3:6.2f} us, "
          f"last stamp {(g[live, :SLOTS - 1].max() - T0) / 1e3:6.2f} us")
for k in range(K):
    g, c = a[k, :, :, 0], a[k, :, :, 1]
    live = g[:, 0] > 0
    g, c = g[live], c[live]
    t0 = g[:, 0].min()
    sm = a[k, :, SLOTS - 1, 1][live].astype(int)
    per_sm = np.bincount(np.bincount(sm, minlength=148))
    print(f"== {names[k]}: {live.sum()} CTAs, kernel span {(g[:, :SLOTS - 1].max() - t0) / 1e3:.2f} us;"
          f" SMs hosting 0,1,2.. CTAs: {per_sm.tolist()}")
    for s, lab in enumerate(labels[k]):
        col = g[:, s]
        ok = col > 0
        if not ok.any():
            continue
        rel = (col[ok] - t0) / 1e3
        dur = (c[ok, s] - c[ok, 0]) / clk
        print(f"   {s} {lab:10s} t[us] min {rel.min():6.2f} med {np.median(rel):6.2f} max {rel.max():6.2f}"
              f" | since start[us] med {np.median(dur):6.2f} max {dur.max():6.2f}")

# the latest CTAs of each kernel (index, phase stamps from the kernel's first start)
for k in range(K):
    g = a[k, :, :, 0]
    idx = np.where(g[:, 0] > 0)[0]
    t0 = g[idx, 0].min()
    last = idx[np.argsort(-g[idx, :SLOTS - 1].max(axis=1))[:6]]
    print(f"# latest {names[k]}: " + "; ".join(
        f"cta {i} sm {int(a[k, i, SLOTS - 1, 1])}: " +
        " ".join(f"{(x - t0) / 1e3:.1f}" for x in g[i, :SLOTS - 1] if x > 0) for i in last))
