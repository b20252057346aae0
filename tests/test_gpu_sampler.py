"""Device cascade sampler (gs_sample_cascades) against the numpy sampler
(the reference's stream, pinned by tests/golden/grid_sampler.npz) and the
oracle's PCG64 restatement, one seed and many seeds per launch."""

import numpy as np
import pytest

from oracle import oracle

pytestmark = pytest.mark.gpu


def _setup(M, lens):
    from paper_2406_14424_b200 import synth
    from paper_2406_14424_b200.cascades import ThresholdGrid
    prof = synth.make_profiles(n_models=M, cost_ratios=tuple(float(4 ** j) for j in range(M)))
    grid = ThresholdGrid({m: tuple(float(x) for x in np.arange(lens[j]) / 100.0)
                          for j, m in enumerate(prof.model_ids)})
    return prof, grid


@pytest.mark.parametrize("M,lens,n", [(3, (100, 100, 100), 2000), (4, (1, 2, 7, 30), 500),
                                      (8, (10,) * 8, 3000), (1, (5,), 10)])
def test_device_sampler_equals_host_sampler(M, lens, n):
    from paper_2406_14424_b200.cascades import sample_cascades, sample_cascades_device
    prof, grid = _setup(M, lens)
    seeds = [0, 1, 17, 123456789]
    outs = sample_cascades_device(prof, grid, n, seeds)
    for seed, out in zip(seeds, outs):
        want = sample_cascades(prof, grid, n, rng_seed=seed)
        assert out.cascades(prof.model_ids) == want
        _, st = oracle.sample_cascades_pcg(lens, n, seed)
        assert out.rng_state == st
        gi = out.grid_index.cpu().numpy()
        th = out.thresholds.cpu().numpy()
        sm = out.stage_model.cpu().numpy()
        ns = out.n_stages.cpu().numpy()
        for i in range(out.count):
            for s in range(ns[i] - 1):
                assert th[i, s] == grid.per_model[prof.model_ids[sm[i, s]]][gi[i, s]]


def test_device_sampler_reference_golden():
    """The reference's own sample_cascades output (grid_sampler.npz)."""
    from conftest import golden
    from paper_2406_14424_b200 import synth
    from paper_2406_14424_b200.cascades import ThresholdGrid, sample_cascades, \
        sample_cascades_device
    g = golden("grid_sampler.npz")
    files = set(g.files)
    # the host sampler is pinned to this golden in test_host; the device
    # sampler must give the host sampler's list for the same inputs
    prof = synth.make_profiles()
    cert, _ = synth.validation_matrices(3, 2000, 0.8, 0)
    from oracle.oracle import grid_values
    grid = ThresholdGrid({m: tuple(grid_values(cert[:, j], 10)) for j, m in
                          enumerate(prof.model_ids)})
    for seed in (0, 5):
        dev = sample_cascades_device(prof, grid, 2000, seed)[0].cascades(prof.model_ids)
        assert dev == sample_cascades(prof, grid, 2000, rng_seed=seed)
    assert files
