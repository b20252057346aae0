"""Time config 4a's front path (1000-level grids, 5 models, N records) on a
k0 slice, or the whole grid: python tools/time_front5.py N K0SLICE"""
import sys
import time
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2406_14424_b200 import synth
from paper_2406_14424_b200.cascades import grid_values
from paper_2406_14424_b200.front5 import Front5, assemble

n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
k0s = int(sys.argv[2]) if len(sys.argv) > 2 else 0
k0b = int(sys.argv[3]) if len(sys.argv) > 3 else 0  # first k0 of the slice
cert, corr = synth.validation_matrices(5, n, 0.8, 7)
grids = [np.array(grid_values(cert[:, j], 1000)) for j in range(5)]
cost1 = np.array([1.0, 4.0, 16.0, 64.0, 256.0])
t = time.perf_counter()
f5 = Front5(cert, corr, grids, cost1)
torch.cuda.synchronize()
print("grid lengths", f5.grid_len, "configs", f5.n_configs, "prepare s", time.perf_counter() - t)
g0 = f5.grid_len[0]
e = g0 if k0s == 0 else min(g0, k0b + k0s)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
ev[0].record()
f5.pass1(k0b, e)
ev[1].record()
nf = f5.select()
ev[2].record()
f5.pass2(k0b, e, cap=0)
ev[3].record()
torch.cuda.synchronize()
p1, sel, p2 = ev[0].elapsed_time(ev[1]), ev[1].elapsed_time(ev[2]), ev[2].elapsed_time(ev[3])
cfg = (e - k0b) / g0 * f5.n_configs
print(f"k0 [{k0b},{e}) configs {cfg:.3e}: pass1 {p1:.1f} ms, select {sel:.2f} ms, pass2 {p2:.1f} ms; "
      f"front accuracies {nf}, front points {len(f5.points()[0])}, front configs {int(f5.points()[2].sum())}; "
      f"{cfg / ((p1 + sel + p2) * 1e-3):.3e} config-evals/s")
torch.cuda.synchronize()
t = time.perf_counter()
f5.select()
torch.cuda.synchronize()
print("select alone s", time.perf_counter() - t)
