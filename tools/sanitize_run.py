"""One small invocation of each kernel family, for compute-sanitizer
(racecheck / synccheck / memcheck).  Shapes are reduced so the tools finish
in minutes; every kernel path of the headline is taken: the four-model
sorted build (g4_sort, g4_gather) and the column-block eval (g4_eval),
the general sweep, the list path, the stage step and gate, Pareto,
quantiles.  Each result is checked against the oracle so a race that
changes a value also fails loudly."""

import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from oracle import oracle  # noqa: E402
from paper_2406_14424_b200 import kernels, synth  # noqa: E402
from paper_2406_14424_b200.cascades import grid_values  # noqa: E402
from paper_2406_14424_b200.gridsweep import GridSweep  # noqa: E402
from paper_2406_14424_b200.stage import GateBatcher, stage_step  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "all"
torch.cuda.set_device(0)
rng = np.random.default_rng(0)
cost1 = np.array([1.0, 4.0, 16.0, 64.0])

if which in ("all", "grid4"):
    c4, k4 = synth.validation_matrices(4, 60_000, 0.8, 1)
    grids4 = [np.array(grid_values(c4[:, j], 40)) for j in range(4)]
    sw4 = GridSweep(c4, k4, grids4, cost1)
    assert sw4.info.fast_path == 2
    res4 = sw4.evaluate(n_correct=True)
    pick = np.unique(rng.integers(0, sw4.n_configs, 400))
    gsm, gthr, gns = oracle.grid_configs(grids4)
    want = oracle.evaluate_encoded(c4, k4, gsm[pick], gthr[pick], gns[pick], cost1)
    assert np.array_equal(res4.accuracy.cpu().numpy()[pick], want[0])
    assert np.array_equal(res4.forward_frac.cpu().numpy()[pick], want[2])
    sw4.pareto(res=res4)
    print("grid4 ok", flush=True)

if which in ("all", "general"):
    c3, k3 = synth.validation_matrices(3, 5000, 0.8, 0)
    grids = [np.array(grid_values(c3[:, j], 20)) for j in range(3)]
    sw = GridSweep(c3, k3, grids, cost1[:3])
    res = sw.evaluate()
    gsm, gthr, gns = oracle.grid_configs(grids)
    want = oracle.evaluate_encoded(c3, k3, gsm, gthr, gns, cost1[:3])
    assert np.array_equal(res.accuracy.cpu().numpy(), want[0])
    print("general ok", flush=True)

if which in ("all", "list"):
    cert = rng.random((3000, 4))
    corr = (rng.random((3000, 4)) < 0.7).astype(np.uint8)
    sm = np.array([[0, 1, 2, -1], [3, -1, -1, -1], [2, 0, 3, 1]] * 50, dtype=np.int32)
    thr = np.array([[0.3, 0.6, 0.0, 0.0], [0.0] * 4, [0.2, 0.9, 0.5, 0.0]] * 50)
    ns = np.array([3, 1, 4] * 50, dtype=np.int32)
    got = kernels.evaluate_encoded(cert, corr, sm, thr, ns, cost1)
    want = oracle.evaluate_encoded(cert, corr, sm, thr, ns, cost1)
    assert all(np.array_equal(a, b) for a, b in zip(got, want))
    print("list ok", flush=True)

if which in ("all", "stage"):
    logits = torch.from_numpy(rng.standard_normal((3000, 1000)).astype(np.float32)).cuda()
    thr_rows = np.full(3000, 0.5)
    out = stage_step(logits, thr_rows, kind="margin")
    cref = oracle.margin_rows(logits.cpu().numpy())
    _, deferred, _, _ = oracle.stage_step(cref, thr_rows)
    assert np.array_equal(out.deferred_idx.cpu().numpy(), deferred)
    stage_step(logits, thr_rows, kind="entropy")
    gb = GateBatcher(torch.from_numpy(rng.random((100, 3))), torch.ones((100, 3), dtype=torch.uint8))
    gb.gate(np.arange(7), np.zeros(7, np.int32), np.full(7, 0.5), np.zeros(7, bool))
    print("stage ok", flush=True)

if which in ("all", "quantile"):
    from paper_2406_14424_b200.cascades import quantiles
    x = np.round(rng.random(20_000), 2)  # ties: long lists in the final select
    qs = [k / 50 for k in range(1, 50)]
    assert np.array_equal(quantiles(x, qs), np.quantile(x, qs))
    y = rng.random(30_000)
    assert np.array_equal(quantiles(y, qs), np.quantile(y, qs))
    print("quantile ok", flush=True)

if which in ("all", "head"):
    from paper_2406_14424_b200.head import head_certainty
    f = torch.randn(700, 256, device="cuda").to(torch.bfloat16)
    w = (torch.randn(300, 256, device="cuda") / 16).to(torch.bfloat16)
    cert, lg = head_certainty(f, w, kind="entropy", logits=True)
    ref = f.double() @ w.double().T
    assert torch.allclose(lg.double(), ref, rtol=1e-5, atol=1e-5)
    head_certainty(f, w, kind="margin")
    print("head ok", flush=True)

if which in ("all", "front5"):
    # config 4a's path (prepare, both passes with the row flags, select)
    # against the materialised five-model sweep + exact front (config 4b's path)
    from paper_2406_14424_b200.front5 import Front5
    from paper_2406_14424_b200.gridsweep import pareto_counts
    c5, k5 = synth.validation_matrices(5, 3000, 0.8, 2)
    grids5 = [np.array(grid_values(c5[:, j], 40)) for j in range(5)]  # g2 > 16: the in-place bound refresh runs
    cost5 = np.array([1.0, 4.0, 16.0, 64.0, 256.0])
    f = Front5(c5, k5, grids5, cost5).front()
    sw5 = GridSweep(c5, k5, grids5, cost5)
    sb = sw5.n_configs - int(np.prod([len(g) for g in grids5[:4]]))
    res5 = sw5.evaluate(sb, sw5.n_configs - sb, n_correct=True)
    idx = pareto_counts(res5.n_correct, res5.mean_cost, sw5.n_rec).cpu().numpy()
    assert np.array_equal(f.index.astype(np.int64), idx)
    assert np.array_equal(f.mean_cost, res5.mean_cost.cpu().numpy()[idx])
    print("front5 ok", flush=True)

torch.cuda.synchronize()
print("sanitize run ok")
