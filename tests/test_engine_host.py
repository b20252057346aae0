"""Host-side replica routing (engine.route) draws the engine's Generator
exactly like a sequence of reference choose_weighted calls (CPU only)."""

import numpy as np

from oracle import oracle
from paper_2406_14424_b200.engine import GearTables, route


def _tables(rng, n_gears=3, zero_stage=None):
    sm, th, rep, cum = [], [], [], []
    for g in range(n_gears):
        k = int(rng.integers(1, 4))
        sm.append(list(range(k)))
        th.append([0.5] * (k - 1) + [None])
        rs, cs = [], []
        for s in range(k):
            n = int(rng.integers(1, 4))
            rs.append(np.arange(n) + 10 * s)
            w = np.round(rng.random(n) * 3, 1)
            if zero_stage is not None and (g, s) == zero_stage:
                w[:] = 0.0
            cs.append(np.cumsum(w))
        rep.append(rs)
        cum.append(cs)
    return GearTables(sm, th, rep, cum)


def test_route_matches_sequential_choose_weighted():
    rng = np.random.default_rng(0)
    for trial in range(40):
        t = _tables(rng, zero_stage=(0, 1) if trial % 3 == 0 else None)
        n = int(rng.integers(0, 200))
        gears = rng.integers(0, len(t.stage_models), n)
        stages = np.array([int(rng.integers(0, len(t.stage_models[g]))) for g in gears],
                          dtype=np.int64)
        seed = int(rng.integers(0, 1 << 30))
        a = np.random.default_rng(seed)
        got = route(t, gears, stages, a)
        b = np.random.default_rng(seed)
        want = [int(t.replicas[g][s][oracle.choose_weighted(t.cum_weights[g][s], b)])
                for g, s in zip(gears, stages)]
        assert list(got) == want
        assert a.random() == b.random()  # generator left in the same state
