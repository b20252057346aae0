"""Config 4b (5 models, 100-level grids, 100k records): build + full eval twice (for ncu)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2406_14424_b200 import synth
from paper_2406_14424_b200.cascades import grid_values
from paper_2406_14424_b200.gridsweep import GridSweep
cert, corr = synth.validation_matrices(5, 100_000, 0.8, 5)
grids = [np.array(grid_values(cert[:, j], 100)) for j in range(5)]
sw = GridSweep(cert, corr, grids, np.array([1.0, 4.0, 16.0, 64.0, 256.0]), build=False)
out = None
for _ in range(2):
    sw.build()
    out = sw.evaluate(out=out)
torch.cuda.synchronize()
print("done", sw.n_configs)
