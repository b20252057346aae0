"""List path (gs_eval_encoded via kernels.evaluate_encoded) vs the reference's
golden outputs and the oracle: bit-exact."""

import numpy as np
import pytest

import golden_inputs as gi
from conftest import golden
from oracle import oracle

pytestmark = pytest.mark.gpu


def _same(a, b):
    for x, y in zip(a, b):
        assert x.shape == y.shape
        assert np.array_equal(x, y), np.flatnonzero(x.reshape(-1) != y.reshape(-1))[:10]


def test_random_problems_bitwise():
    from paper_2406_14424_b200 import kernels
    g = golden("kernels.npz")
    rng = np.random.default_rng(12345)
    for t in range(5):
        args = gi.random_problem(rng)
        got = kernels.evaluate_encoded(*args)
        _same(got, (g[f"rp{t}_acc"], g[f"rp{t}_cost"], g[f"rp{t}_frac"]))


def test_bench_problem_bitwise():
    from paper_2406_14424_b200 import kernels
    g = golden("kernels.npz")
    got = kernels.evaluate_encoded(*gi.bench_problem(4000, 6, 200, 0))
    _same(got, (g["bench_acc"], g["bench_cost"], g["bench_frac"]))


def test_c1_fixtures_bitwise():
    from paper_2406_14424_b200 import kernels
    g = golden("c1.npz")
    for i, fx in enumerate(gi.c1_fixtures()):
        sm, thr, ns = gi.encode(fx["cascades"], fx["mids"])
        got = kernels.evaluate_encoded(g[f"f{i}_cert"], g[f"f{i}_corr"], sm, thr, ns,
                                       np.asarray(fx["cost1"], dtype=np.float64))
        _same(got, (g[f"f{i}_acc"], g[f"f{i}_cost"], g[f"f{i}_frac"]))


def test_known_answers():
    from paper_2406_14424_b200 import kernels
    rng = np.random.default_rng(1)
    acc, cost, frac = kernels.evaluate_encoded(
        rng.random((10, 2)), np.array([[1, 0]] * 10, dtype=np.uint8), np.array([[0]]),
        np.zeros((1, 1)), np.array([1]), np.array([100.0, 200.0]))
    assert acc[0] == 1.0 and cost[0] == 100.0 and frac[0, 0] == 1.0
    # inclusive boundary: cert == thr stops
    acc, cost, frac = kernels.evaluate_encoded(
        np.array([[0.5, 0.5]]), np.array([[1, 0]], dtype=np.uint8), np.array([[0, 1]]),
        np.array([[0.5, 0.0]]), np.array([2]), np.array([5000.0, 20000.0]))
    assert frac[0, 1] == 0.0 and acc[0] == 1.0
    # empty cascade list keeps the reference's shapes
    acc, cost, frac = kernels.evaluate_encoded(np.zeros((3, 2)), np.zeros((3, 2)),
                                               np.zeros((0, 3)), np.zeros((0, 3)),
                                               np.zeros(0), np.ones(2))
    assert acc.shape == (0,) and frac.shape == (0, 3)


@pytest.mark.parametrize("n_rec,n_models,n_casc,max_len", [
    (1, 1, 1, 1), (17, 3, 5, 3), (1000, 6, 777, 6), (4099, 16, 300, 16), (50_000, 4, 2000, 4),
    (3, 9, 1, 9)])
def test_random_vs_oracle(n_rec, n_models, n_casc, max_len):
    from paper_2406_14424_b200 import kernels
    rng = np.random.default_rng(n_rec * 7 + n_models)
    args = gi.random_problem(rng, n_rec=n_rec, n_models=n_models, n_casc=n_casc,
                             max_len=max_len)
    _same(kernels.evaluate_encoded(*args), oracle.evaluate_encoded(*args, n_threads=8))


def test_unaligned_device_views():
    """Offset views defeat 16-byte alignment: the cooperative-copy path."""
    import torch
    from paper_2406_14424_b200 import kernels
    rng = np.random.default_rng(3)
    cert, corr, sm, thr, ns, cost1 = gi.random_problem(rng, n_rec=3001, n_models=3, n_casc=40,
                                                       max_len=3)
    dev = torch.device("cuda")
    big = torch.zeros(cert.size + 1, dtype=torch.float64, device=dev)
    big[1:] = torch.from_numpy(cert.reshape(-1)).to(dev)
    cbig = torch.zeros(corr.size + 3, dtype=torch.uint8, device=dev)
    cbig[3:] = torch.from_numpy(corr.reshape(-1)).to(dev)
    t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a)).to(dev, dt)
    out = kernels.evaluate_encoded_device(big[1:].view(3001, 3), cbig[3:].view(3001, 3),
                                          t(sm, torch.int32), t(thr, torch.float64),
                                          t(ns, torch.int32), t(cost1, torch.float64))
    _same([o.cpu().numpy() for o in out], oracle.evaluate_encoded(cert, corr, sm, thr, ns, cost1))


def test_bad_model_index_raises():
    from paper_2406_14424_b200 import kernels
    with pytest.raises(IndexError):
        kernels.evaluate_encoded(np.zeros((2, 2)), np.zeros((2, 2)), np.array([[0, 2]]),
                                 np.zeros((1, 2)), np.array([2]), np.ones(2))


def test_long_cascades_vs_oracle():
    """Encoded cascades of 17..40 stages (40 models): the 32- and 64-stage
    instances of the list kernel."""
    from paper_2406_14424_b200 import kernels
    rng = np.random.default_rng(3)
    n_models, n_rec = 40, 3000
    cert = rng.random((n_rec, n_models))
    corr = (rng.random((n_rec, n_models)) < 0.6).astype(np.uint8)
    for L in (20, 40):
        n_casc = 50
        sm = np.full((n_casc, L), -1, dtype=np.int32)
        thr = np.zeros((n_casc, L))
        ns = rng.integers(1, L + 1, n_casc).astype(np.int32)
        for c in range(n_casc):
            sm[c, :ns[c]] = rng.choice(n_models, ns[c], replace=False)
            thr[c, :ns[c] - 1] = rng.random(ns[c] - 1) * 0.3 + 0.7
        cost1 = rng.uniform(1, 100, n_models)
        got = kernels.evaluate_encoded(cert, corr, sm, thr, ns, cost1)
        want = oracle.evaluate_encoded(cert, corr, sm, thr, ns, cost1)
        for a, b in zip(got, want):
            assert np.array_equal(a, b)
