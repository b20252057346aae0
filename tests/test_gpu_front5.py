"""Config 4a's Pareto-front path (gs_front5.cu) against the materialised
sweep: every config of the full five-model cascade scored by the grid path
(gs_sweep5.cu, itself bit-exact against the oracle walk), its exact front
taken by gs_pareto_counts -- the same index set, costs, accuracies and
forward fractions, bit for bit; also sharded by k0 with the MIN reduction
of the per-accuracy costs, as the multi-GPU run does."""

import numpy as np
import pytest
import torch

from oracle import oracle

pytestmark = pytest.mark.gpu


def _case(n_rec, levels, seed, ties=False):
    from paper_2406_14424_b200 import synth
    from paper_2406_14424_b200.cascades import grid_values
    cert, corr = synth.validation_matrices(5, n_rec, 0.8, seed)
    if ties:
        cert = np.round(cert, 2)
    grids = [np.array(grid_values(cert[:, j], levels)) for j in range(5)]
    cost1 = np.array([1.0, 4.0, 16.0, 64.0, 256.0])
    return cert, corr, grids, cost1


def _reference_front(cert, corr, grids, cost1):
    from paper_2406_14424_b200.gridsweep import GridSweep, pareto_counts
    sw = GridSweep(cert, corr, grids, cost1)
    sb = sw.n_configs - int(np.prod([len(g) for g in grids[:4]]))
    res = sw.evaluate(sb, sw.n_configs - sb, n_correct=True)
    idx = pareto_counts(res.n_correct, res.mean_cost, sw.n_rec).cpu().numpy()
    return (idx, res.accuracy.cpu().numpy()[idx], res.mean_cost.cpu().numpy()[idx],
            res.forward_frac.cpu().numpy()[idx])


@pytest.mark.parametrize("n_rec,levels,ties", [(4000, 12, False), (6000, 25, True),
                                               (20_000, 40, False)])
def test_front_equals_materialised_sweep(n_rec, levels, ties):
    from paper_2406_14424_b200.front5 import Front5
    cert, corr, grids, cost1 = _case(n_rec, levels, n_rec + levels, ties)
    want = _reference_front(cert, corr, grids, cost1)
    f5 = Front5(cert, corr, grids, cost1)
    f = f5.front()
    assert np.array_equal(f.index.astype(np.int64), want[0])
    assert np.array_equal(f.accuracy, want[1])
    # the per-point summary (what the 1000-level run reports): tie counts and
    # smallest index of each distinct front point
    a, c, ties, mi = f5.points()
    pts = {}
    for i, nc, cc in zip(f.index, f.n_correct, f.mean_cost):
        k = (int(nc), float(cc))
        pts.setdefault(k, []).append(int(i))
    assert sorted(pts) == sorted(zip(a.tolist(), c.tolist()))
    for nc, cc, t, m in zip(a, c, ties, mi):
        assert int(t) == len(pts[(int(nc), float(cc))]) and int(m) == min(pts[(int(nc), float(cc))])
    assert np.array_equal(f.mean_cost, want[2])
    assert np.array_equal(f.forward_frac, want[3])
    # and the oracle walk on the front configs themselves (front5's decode =
    # gridsweep's decode of the full cascade's block)
    from paper_2406_14424_b200.gridsweep import GridSweep
    sw = GridSweep(cert, corr, grids, cost1, build=False)
    sb = sw.n_configs - int(np.prod([len(g) for g in grids[:4]]))
    sm, thr, ns = (t.cpu().numpy() for t in sw.decode(sb + f.index.astype(np.int64)))
    dsm, dthr, dns = f5.decode(f.index)
    assert np.array_equal(dsm, sm) and np.array_equal(dthr, thr) and np.array_equal(dns, ns)
    w = oracle.evaluate_encoded(cert, corr, sm, thr, ns, cost1, n_threads=8)
    assert np.array_equal(w[0], f.accuracy) and np.array_equal(w[1], f.mean_cost)


def test_sharded_by_k0_with_min_reduction():
    """Four k0 shards, each its own pass 1; mincost reduced with MIN (what
    the NCCL all-reduce does across ranks); each shard's pass 2 emits its
    slice of the front: the union is the single-device front."""
    from paper_2406_14424_b200.front5 import Front5, assemble
    cert, corr, grids, cost1 = _case(8000, 20, 3)
    whole = Front5(cert, corr, grids, cost1).front()
    g0 = len(grids[0])
    cuts = np.linspace(0, g0, 5).astype(int)
    shards = [Front5(cert, corr, grids, cost1) for _ in range(4)]
    for s, (b, e) in zip(shards, zip(cuts[:-1], cuts[1:])):
        s.pass1(b, e)
    red = torch.stack([s.mincost() for s in shards]).min(dim=0).values
    parts = []
    for s, (b, e) in zip(shards, zip(cuts[:-1], cuts[1:])):
        s.mincost().copy_(red)
        s.select()
        parts.append(s.pass2(b, e))
    idx = torch.cat([p[0] for p in parts])
    cost = torch.cat([p[1] for p in parts])
    cnt = torch.cat([p[2] for p in parts])
    f = assemble(idx, cost, cnt, 8000, whole.n_configs)
    assert np.array_equal(f.index, whole.index)
    assert np.array_equal(f.mean_cost, whole.mean_cost)


def test_config4b_shape_front():
    """100-level grids over 100k records: the 1.03e8 full-cascade configs'
    front, against the materialised sweep (the config-4b path)."""
    from paper_2406_14424_b200.front5 import Front5
    cert, corr, grids, cost1 = _case(100_000, 100, 5)
    want = _reference_front(cert, corr, grids, cost1)
    f = Front5(cert, corr, grids, cost1).front()
    assert np.array_equal(f.index.astype(np.int64), want[0])
    assert np.array_equal(f.mean_cost, want[2])
    assert np.array_equal(f.forward_frac, want[3])
