"""Locate general-path (M=4) mismatches: per structure, first bad config."""
import sys
import numpy as np
sys.path.insert(0, ".")
from oracle import oracle
from paper_2406_14424_b200.gridsweep import GridSweep, structures

for glen in [(255, 3, 200, 2), (255, 3, 50, 2), (150, 3, 200, 2), (161, 3, 20, 2), (255, 1, 1, 1),
             (200, 5, 5, 2), (130, 5, 5, 2)]:
    rng = np.random.default_rng(sum(glen))
    n = 5000
    cert = rng.random((n, 4))
    corr = (rng.random((n, 4)) < 0.6).astype(np.uint8)
    grids = [np.concatenate([[0.0], np.sort(rng.random(g - 1))]) for g in glen]
    cost1 = np.array([1.0, 3.0, 9.0, 27.0])
    sw = GridSweep(cert, corr, grids, cost1)
    res = sw.evaluate(n_correct=True)
    acc = res.accuracy.cpu().numpy()
    frac = res.forward_frac.cpu().numpy()
    bad = []
    for models, b, cnt in structures(4, sw.grid_len):
        pick = np.unique(np.linspace(b, b + cnt - 1, min(cnt, 50)).astype(np.int64))
        sm, thr, ns = (t.cpu().numpy() for t in sw.decode(pick))
        want = oracle.evaluate_encoded(cert, corr, sm, thr, ns, cost1, n_threads=8)
        ok_a = acc[pick] == want[0]
        ok_f = np.all(frac[pick] == want[2], axis=1)
        if not (ok_a.all() and ok_f.all()):
            i = int(np.flatnonzero(~(ok_a & ok_f))[0])
            bad.append((models, int(pick[i] - b), float(acc[pick[i]]), float(want[0][i]),
                        frac[pick[i]].tolist(), want[2][i].tolist()))
    print(glen, "fast" if sw.info.fast_path else ("walk" if sw.info.eval_launches == 2 else "general"),
          "OK" if not bad else f"{len(bad)} bad structures")
    for x in bad[:6]:
        print("   ", x)
