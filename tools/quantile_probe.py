"""Device time of gs_quantiles (99 quantiles of a 1M-value column, the
config-3 / 4b threshold-grid shape): CUDA events around back-to-back calls."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2406_14424_b200.cascades import quantiles

rng = np.random.default_rng(0)
qs = [k / 100 for k in range(1, 100)]
for name, x in (("uniform", rng.random(1_000_000)),
                ("margins", np.abs(rng.standard_normal(1_000_000)) / 4),
                ("ties", np.round(rng.random(1_000_000), 2))):
    t = torch.from_numpy(x).cuda()
    got = quantiles(t, qs)
    assert np.array_equal(got, np.quantile(x, qs)), name
    for _ in range(3):
        quantiles(t, qs)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    a.record()
    for _ in range(reps):
        quantiles(t, qs)
    b.record()
    torch.cuda.synchronize()
    print(f"{name:8s} 1M values, 99 quantiles: {a.elapsed_time(b) / reps * 1e3:8.1f} us per call (events, "
          f"includes the host call and its H2D of the qs)", flush=True)
