"""SP1-shape list path (sample_cascades over the config-2 100-level grids x
1M records, gs_eval_encoded, device resident): median of 10 launches by CUDA
events, checked against the first.  python tools/list_probe.py"""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2406_14424_b200 import kernels  # noqa: E402
from paper_2406_14424_b200.cascades import ThresholdGrid, encode_cascades, sample_cascades  # noqa: E402

profiles, cert, corr, grids, cost1 = bench.workload(seed=0)
grid = ThresholdGrid({m: tuple(float(x) for x in grids[j]) for j, m in enumerate(profiles.model_ids)})
sm, thr, ns = encode_cascades(sample_cascades(profiles, grid, 2000, rng_seed=0), profiles)
d = [torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in (cert, corr, sm, thr, ns, cost1)]
ref = kernels.evaluate_encoded_device(*d)
ts = []
for _ in range(10):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    r = kernels.evaluate_encoded_device(*d)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
same = all(torch.equal(x, y) for x, y in zip(r, ref))
print(f"sp1 list path: {len(ns)} cascades x {cert.shape[0]} records: {np.median(ts):.3f} ms same={same}")
