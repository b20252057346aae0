"""The TORCH_LIBRARY operators (csrc/gs_torch_ops.cpp): registration on CPU,
and on the GPU each op against the ctypes-bound library / the oracle."""

import numpy as np
import pytest
import torch

from oracle import oracle


def test_ops_library_registers_every_op():
    from paper_2406_14424_b200 import torch_ops
    ops = torch_ops.load()
    for name in torch_ops.OPS:
        schema = str(getattr(ops, name).default._schema)
        assert schema.startswith(f"gearserve_b200::{name}(")
    with pytest.raises((NotImplementedError, RuntimeError)):  # no CPU kernel: no fallback
        ops.certainty(torch.zeros(2, 3), 0)


@pytest.mark.gpu
def test_ops_match_the_library_and_the_oracle():
    from paper_2406_14424_b200 import kernels, synth, torch_ops
    from paper_2406_14424_b200.cascades import certainty_rows, grid_values, quantiles
    from paper_2406_14424_b200.gridsweep import GridSweep
    ops = torch_ops.load()
    rng = np.random.default_rng(5)
    cert = rng.random((3000, 4))
    corr = (rng.random((3000, 4)) < 0.7).astype(np.uint8)
    sm = np.array([[0, 1, 2, -1], [3, -1, -1, -1], [2, 0, 3, 1]], dtype=np.int32)
    thr = np.array([[0.3, 0.6, 0.0, 0.0], [0.0] * 4, [0.2, 0.9, 0.5, 0.0]])
    ns = np.array([3, 1, 4], dtype=np.int32)
    cost1 = np.array([1.0, 4.0, 16.0, 64.0])
    d = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()  # noqa: E731
    got = ops.evaluate_encoded(d(cert), d(corr), d(sm), d(thr), d(ns), d(cost1))
    want = oracle.evaluate_encoded(cert, corr, sm, thr, ns, cost1)
    for a, b in zip(got, want):
        assert np.array_equal(a.cpu().numpy(), b)
    # the grid sweep (headline four-model fast path) vs GridSweep, and its front
    c4, k4 = synth.validation_matrices(4, 20_000, 0.8, 1)
    grids = [np.array(grid_values(c4[:, j], 30)) for j in range(4)]
    acc, cost, frac, nc = ops.grid_sweep(d(c4), d(k4), d(np.concatenate(grids)), [len(g) for g in grids],
                                         d(cost1))
    res = GridSweep(c4, k4, grids, cost1).evaluate(n_correct=True)
    assert torch.equal(acc, res.accuracy) and torch.equal(cost, res.mean_cost)
    assert torch.equal(frac, res.forward_frac) and torch.equal(nc.view(torch.int32), res.n_correct.view(torch.int32))
    front = ops.pareto_counts(nc, cost, 20_000).cpu().numpy()
    assert np.array_equal(front, np.flatnonzero(oracle.pareto_keep(acc.cpu().numpy(), cost.cpu().numpy())))
    # certainty (margin, the reference's) and quantiles
    logits = torch.randn(500, 10, dtype=torch.float64, device="cuda")
    assert torch.equal(ops.certainty(logits, 0), certainty_rows(logits, kind="margin"))
    col = d(c4)[:, 2]
    assert np.array_equal(ops.quantiles(col, [0.1, 0.5, 0.9]).cpu().numpy(), quantiles(col, [0.1, 0.5, 0.9]))
    with pytest.raises(ValueError):
        ops.evaluate_encoded(d(cert), d(corr[:10]), d(sm), d(thr), d(ns), d(cost1))
    # the tensor-core head
    from paper_2406_14424_b200.head import head_certainty
    f = torch.randn(300, 128, device="cuda").to(torch.bfloat16)
    w = torch.randn(50, 128, device="cuda").to(torch.bfloat16)
    b = torch.randn(50, device="cuda")
    assert torch.equal(ops.head_certainty(f, w, b, 2), head_certainty(f, w, b, kind="entropy"))
