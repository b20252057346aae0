"""Device quantiles (gs_quantiles) vs np.quantile (numpy "linear"), bit for
bit, and the threshold grid built from them vs the reference golden."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _q(levels):
    return [k / levels for k in range(1, levels)]


@pytest.mark.parametrize("n,kind", [(1, "rand"), (2, "rand"), (3, "ties"), (10, "rand"),
                                     (1000, "ties"), (4097, "rand"), (100_000, "bands"),
                                     (1_000_000, "rand")])
def test_quantiles_equal_numpy(n, kind):
    from paper_2406_14424_b200.cascades import quantiles
    rng = np.random.default_rng(n)
    if kind == "rand":
        x = rng.random(n)
    elif kind == "ties":
        x = np.round(rng.random(n), 1)
    else:
        x = np.where(rng.random(n) < 0.8, rng.uniform(0.6, 0.95, n), rng.uniform(0.0, 0.3, n))
    qs = sorted(set(_q(100) + _q(7) + [0.0, 1.0, 0.5, 0.999999]))
    got = quantiles(x, qs)
    want = np.quantile(x, qs)
    assert np.array_equal(got, want)


def test_quantiles_of_a_strided_device_column_and_special_values():
    from paper_2406_14424_b200.cascades import quantiles
    rng = np.random.default_rng(3)
    m = rng.random((5000, 4))
    m[::7, 2] = -m[::7, 2]
    m[10, 2] = -0.0
    t = torch.from_numpy(m).cuda()
    for j in range(4):
        assert np.array_equal(quantiles(t[:, j], _q(10)), np.quantile(m[:, j], _q(10)))
    x = rng.random(100)
    x[17] = np.nan
    assert np.all(np.isnan(quantiles(x, [0.1, 0.5])))
    x = np.array([1.0, np.inf, -np.inf, 2.0])
    assert np.array_equal(quantiles(x, [0.0, 0.4, 1.0]), np.quantile(x, [0.0, 0.4, 1.0]),
                          equal_nan=True)  # inf - inf: NaN in both
    with pytest.raises(ValueError):
        quantiles(np.arange(4.0), [1.5])


def test_threshold_grid_equals_reference_golden_on_synth():
    from conftest import golden
    from paper_2406_14424_b200 import cascades as gc
    from paper_2406_14424_b200 import synth
    g = golden("grid_sampler.npz")
    p3 = synth.make_profiles()
    va = synth.make_validation_arrays(p3, 400, 0.8, seed=0)
    grid = gc.build_threshold_grid(va, p3, levels=10)
    for m in p3.model_ids:
        assert np.array_equal(np.array(grid.per_model[m]), g[f"synth_grid_{m}"])


@pytest.mark.parametrize("kind", ["rand", "ties"])
def test_many_quantiles_in_rounds(kind):
    """1000-level grids (config 4a) need 999 quantiles: the select runs them in
    rounds of 255 over the same keys."""
    from paper_2406_14424_b200.cascades import grid_values, quantiles
    rng = np.random.default_rng(11)
    x = rng.random(200_000) if kind == "rand" else np.round(rng.random(200_000), 3)
    qs = _q(1000)
    assert np.array_equal(quantiles(x, qs), np.quantile(x, qs))
    g = grid_values(x, 1000)
    assert g == tuple(sorted({0.0} | {float(v) for v in np.quantile(x, qs)}))
