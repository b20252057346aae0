"""Host logic of config 4a's sharding (no GPU): front5.k0_cuts splits k0
= 0..g0 into contiguous per-rank ranges of about equal modelled work."""
import numpy as np
import pytest

from paper_2406_14424_b200.front5 import k0_cuts


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_k0_cuts_cover_and_balance(world):
    rng = np.random.default_rng(1)
    x = rng.random(100_000)
    g = np.concatenate([[0.0], np.quantile(x, np.arange(1, 1000) / 1000)])
    cuts = k0_cuts(x, g, world)
    assert cuts.shape == (world + 1,) and cuts[0] == 0 and cuts[-1] == g.size
    assert np.all(np.diff(cuts) > 0)
    b0 = np.searchsorted(g, x, side="right")
    r = np.cumsum(np.bincount(b0, minlength=g.size + 1))[: g.size]
    w = 1.0 + 2.0 * r / x.size
    per = np.array([w[cuts[i]:cuts[i + 1]].sum() for i in range(world)])
    assert per.max() <= 1.01 * per.mean() + w.max()
    if world > 1:  # later k0 cost more: the last rank gets fewer of them
        assert cuts[-1] - cuts[-2] < cuts[1] - cuts[0]


def test_k0_cuts_more_ranks_than_k0():
    cuts = k0_cuts(np.array([0.5, 0.7]), np.array([0.0, 0.6]), 4)
    assert cuts[0] == 0 and cuts[-1] == 2 and np.all(np.diff(cuts) >= 0)
