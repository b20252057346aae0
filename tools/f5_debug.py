import sys
import numpy as np
sys.path.insert(0, "/root/repo/tests"); sys.path.insert(0, "/root/repo")
from test_gpu_front5 import _case, _reference_front
from paper_2406_14424_b200.front5 import Front5
cert, corr, grids, cost1 = _case(4000, 12, 4012, False)
want = _reference_front(cert, corr, grids, cost1)
f = Front5(cert, corr, grids, cost1).front()
got = f.index.astype(np.int64)
print("want", len(want[0]), "got", len(got))
miss = np.setdiff1d(want[0], got); extra = np.setdiff1d(got, want[0])
print("missing", len(miss), "extra", len(extra))
gl = [len(g) for g in grids]
for i in miss[:10]:
    k3 = i % gl[3]; r = i // gl[3]; k2 = r % gl[2]; r //= gl[2]; k1 = r % gl[1]; k0 = r // gl[1]
    j = np.flatnonzero(want[0] == i)[0]
    print("miss", i, (k0, k1, k2, k3), "acc", want[1][j], "cost", want[2][j])
