import sys, ctypes, numpy as np, torch
sys.path.insert(0, ".")
from paper_2406_14424_b200 import synth, _lib
from paper_2406_14424_b200.cascades import grid_values
from paper_2406_14424_b200.front5 import Front5
lib = _lib.load()
n = 100_000
cert, corr = synth.validation_matrices(5, n, 0.8, 7)
grids = [np.array(grid_values(cert[:, j], 1000)) for j in range(5)]
f5 = Front5(cert, corr, grids, np.array([1.0, 4.0, 16.0, 64.0, 256.0]))
st = (ctypes.c_ulonglong * 8)()
lib.gs_f5_stats(st)
f5.pass1(0, 1000); torch.cuda.synchronize(); f5.select(); f5.pass2(0, 1000, cap=0); torch.cuda.synchronize()
lib.gs_f5_stats(st)
print("rows total 1e9; pass1 scored/live/reach/hit:", list(st)[:4], " pass2:", list(st)[4:])
