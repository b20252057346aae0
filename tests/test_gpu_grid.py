"""Grid path (gs_grid_build/eval/decode + gs_pareto_counts) vs the reference
golden (config 1) and the oracle walk over the enumerated configs."""

import os

import numpy as np
import pytest

from conftest import golden
from oracle import oracle

pytestmark = pytest.mark.gpu


def _sweep(cert, corr, grids, cost1):
    from paper_2406_14424_b200.gridsweep import GridSweep
    sw = GridSweep(cert, corr, grids, cost1)
    res = sw.evaluate(n_correct=True)
    return sw, [t.cpu().numpy() for t in (res.accuracy, res.mean_cost, res.forward_frac,
                                          res.n_correct)]


def test_config1_full_grid_bitwise():
    from paper_2406_14424_b200 import synth
    g = golden("config1.npz")
    cert, corr = synth.validation_matrices(3, 10_000, 0.8, 0)
    grids = [g["grid0"], g["grid1"], g["grid2"]]
    sw, (acc, cost, frac, nc) = _sweep(cert, corr, grids, g["cost1"])
    assert sw.n_configs == 10_303
    assert np.array_equal(acc, g["acc"])
    assert np.array_equal(cost, g["cost"])
    assert np.array_equal(frac, g["frac"])
    assert np.array_equal(nc / 10_000, g["acc"])


def _random_case(rng, n_rec, n_models, levels, ties=False):
    if ties:
        cert = np.round(rng.random((n_rec, n_models)), 1)
    else:
        cert = rng.random((n_rec, n_models))
    corr = (rng.random((n_rec, n_models)) < 0.6).astype(np.uint8)
    grids = []
    for j in range(n_models):
        q = np.quantile(cert[:, j], np.arange(1, levels) / levels)
        grids.append(np.array(sorted({0.0} | {float(x) for x in q})))
    cost1 = rng.uniform(100, 5000, n_models)
    return cert, corr, grids, cost1


@pytest.mark.parametrize("n_rec,n_models,levels,ties", [
    (1, 1, 2, False), (7, 2, 3, False), (500, 3, 10, True), (3000, 4, 12, False),
    (2000, 5, 6, True), (900, 6, 4, False), (300, 8, 3, True), (65_537, 2, 50, False)])
def test_random_grids_vs_oracle(n_rec, n_models, levels, ties):
    rng = np.random.default_rng(n_rec + 31 * n_models)
    cert, corr, grids, cost1 = _random_case(rng, n_rec, n_models, levels, ties)
    sw, (acc, cost, frac, nc) = _sweep(cert, corr, grids, cost1)
    sm, thr, ns = oracle.grid_configs(grids)
    want = oracle.evaluate_encoded(cert, corr, sm, thr, ns, cost1, n_threads=8)
    assert np.array_equal(acc, want[0])
    assert np.array_equal(cost, want[1])
    assert np.array_equal(frac, want[2])
    # decode reproduces the enumeration
    dsm, dthr, dns = (t.cpu().numpy() for t in sw.decode(np.arange(sw.n_configs)))
    assert np.array_equal(dsm, sm) and np.array_equal(dthr, thr) and np.array_equal(dns, ns)
    # exact Pareto front vs the restated pareto_filter
    idx, _ = sw.pareto()
    keep = oracle.pareto_keep(want[0], want[1])
    assert np.array_equal(idx.cpu().numpy(), np.flatnonzero(keep))


@pytest.mark.parametrize("n_models", [4, 5])
def test_config_ranges_equal_full_sweep(n_models):
    """Ranges of the enumeration (crossing the full cascade's start, inside
    one of its (k0, k1) blocks, ...) score exactly like the full sweep."""
    rng = np.random.default_rng(9)
    cert, corr, grids, cost1 = _random_case(rng, 4000, n_models, 9)
    from paper_2406_14424_b200.gridsweep import GridSweep
    sw = GridSweep(cert, corr, grids, cost1)
    full = sw.evaluate(n_correct=True)
    n = sw.n_configs
    sb = n - int(np.prod([len(g) for g in grids[:-1]]))  # first config of the full cascade
    if n_models == 5:  # the full-cascade kernel's whole answer, against the oracle
        sm, thr, ns = oracle.grid_configs(grids)
        pick = np.sort(rng.choice(np.arange(sb, n), size=64, replace=False))
        want = oracle.evaluate_encoded(cert, corr, sm[pick], thr[pick], ns[pick], cost1, n_threads=8)
        assert np.array_equal(full.accuracy.cpu().numpy()[pick], want[0])
        assert np.array_equal(full.mean_cost.cpu().numpy()[pick], want[1])
        assert np.array_equal(full.forward_frac.cpu().numpy()[pick], want[2])
    for begin, count in ((0, 1), (3, 100), (n - 7, 7), (123, n - 200), (5, 3),
                         (sb - 5, 20), (sb + 17, 101), (sb + 64 * 8 + 3, 700)):
        begin = min(begin, n - 1)
        count = min(count, n - begin)
        part = sw.evaluate(begin, count)
        assert np.array_equal(part.accuracy.cpu().numpy(),
                              full.accuracy[begin:begin + count].cpu().numpy())
        assert np.array_equal(part.forward_frac.cpu().numpy(),
                              full.forward_frac[begin:begin + count].cpu().numpy())
        assert np.array_equal(part.mean_cost.cpu().numpy(),
                              full.mean_cost[begin:begin + count].cpu().numpy())


@pytest.mark.parametrize("n_models", [2, 4])
def test_heavy_tie_cell_overflow_fallback(n_models):
    """> 65535 records in one table cell: the packed 16-bit histogram flags
    the overflow and the f32 fallback pass must give the exact counts."""
    rng = np.random.default_rng(17)
    n = 70_000
    cert = np.full((n, n_models), 0.5)
    cert[:5000] = np.round(rng.random((5000, n_models)), 1)  # a few other cells
    corr = (rng.random((n, n_models)) < 0.5).astype(np.uint8)
    grids = [np.array([0.0, 0.25, 0.5, 0.75])] * n_models
    cost1 = np.arange(1, n_models + 1, dtype=np.float64) * 100.0
    sw, (acc, cost, frac, nc) = _sweep(cert, corr, grids, cost1)
    sm, thr, ns = oracle.grid_configs(grids)
    want = oracle.evaluate_encoded(cert, corr, sm, thr, ns, cost1, n_threads=8)
    assert np.array_equal(acc, want[0]) and np.array_equal(cost, want[1])
    assert np.array_equal(frac, want[2])
    # a second build on the same workspace (histogram re-zeroed by the first)
    sw.build()
    res = sw.evaluate()
    assert np.array_equal(res.accuracy.cpu().numpy(), want[0])


@pytest.mark.parametrize("n", [1, 2, 3, 7, 100, 997, 4096, 16000])
def test_count_division_exhaustive(n):
    """Every forward count 0..n and many correct counts appear once as a
    config output: the kernel's FMA-corrected division must equal IEEE x/n
    for all of them (the oracle divides with C `/`)."""
    rng = np.random.default_rng(n)
    vals = np.arange(1, n + 1) / n
    cert = np.stack([rng.permutation(vals), rng.random(n)], axis=1)
    corr = (rng.random((n, 2)) < 0.5).astype(np.uint8)
    grids = [np.sort(vals), np.array([0.0])]
    cost1 = np.array([3.0, 7.0])
    sw, (acc, cost, frac, nc) = _sweep(cert, corr, grids, cost1)
    sm, thr, ns = oracle.grid_configs(grids)
    want = oracle.evaluate_encoded(cert, corr, sm, thr, ns, cost1)
    assert np.array_equal(frac, want[2]) and np.array_equal(acc, want[0])
    assert np.array_equal(cost, want[1])
    reach = np.rint(frac[:, 1] * n).astype(np.int64)
    assert set(range(n)) <= set(reach.tolist()) | {0}


def test_negative_singleton_certainty_bins_below_zero():
    """Singleton scores can be negative (cascades.certainty returns the score):
    such records sit below grid value 0 and forward at every threshold."""
    cert = np.array([[-0.5, 0.2], [0.3, 0.9], [0.0, 0.1]])
    corr = np.array([[1, 0], [0, 1], [1, 1]], dtype=np.uint8)
    grids = [np.array([0.0, 0.3]), np.array([0.0, 0.5])]
    sw, (acc, cost, frac, nc) = _sweep(cert, corr, grids, np.array([1.0, 10.0]))
    sm, thr, ns = oracle.grid_configs(grids)
    want = oracle.evaluate_encoded(cert, corr, sm, thr, ns, np.array([1.0, 10.0]))
    assert np.array_equal(acc, want[0]) and np.array_equal(frac, want[2])


def test_config2_shape_sampled_configs():
    """Config 2 at full size (1M records, 4 models, 100-level grids): a fixed
    sample of configs from every structure matches the oracle walk exactly,
    and the front is a fixed point of the Pareto filter."""
    from paper_2406_14424_b200 import synth
    from paper_2406_14424_b200.cascades import grid_values
    from paper_2406_14424_b200.gridsweep import GridSweep, pareto_counts, structures
    cert, corr = synth.validation_matrices(4, 1_000_000, 0.8, 0)
    grids = [np.array(grid_values(cert[:, j], 100)) for j in range(4)]
    cost1 = np.array([2000.0, 8000.0, 32000.0, 128000.0])
    sw = GridSweep(cert, corr, grids, cost1)
    assert sw.n_configs == sum(n for _, _, n in structures(4, [len(x) for x in grids]))
    res = sw.evaluate(n_correct=True)
    rng = np.random.default_rng(0)
    pick = []
    for _, b, n in structures(4, sw.grid_len):
        pick.extend(sorted(set(rng.integers(b, b + n, size=min(n, 40)).tolist())))
    pick = np.array(pick)
    sm, thr, ns = oracle.grid_configs(grids)  # full enumeration, 1M rows
    want = oracle.evaluate_encoded(cert, corr, sm[pick], thr[pick], ns[pick], cost1,
                                   n_threads=8)
    assert np.array_equal(res.accuracy.cpu().numpy()[pick], want[0])
    assert np.array_equal(res.mean_cost.cpu().numpy()[pick], want[1])
    assert np.array_equal(res.forward_frac.cpu().numpy()[pick], want[2])
    idx, _ = sw.pareto(res=res)
    again = pareto_counts(res.n_correct[idx], res.mean_cost[idx], sw.n_rec)
    assert np.array_equal(idx[again].cpu().numpy(), idx.cpu().numpy())
    keep = oracle.pareto_keep(res.accuracy.cpu().numpy(), res.mean_cost.cpu().numpy())
    assert np.array_equal(idx.cpu().numpy(), np.flatnonzero(keep))


@pytest.mark.parametrize("n_rec,glen,ties", [
    (1, (1, 1, 1, 1), False), (5, (2, 3, 1, 4), False), (400, (7, 1, 9, 3), True),
    (2500, (12, 5, 8, 6), False), (3000, (20, 20, 20, 2), True), (1500, (3, 30, 2, 9), False),
    (70_000, (33, 17, 40, 5), False)])
def test_four_model_uneven_grids_vs_oracle(n_rec, glen, ties):
    """The four-model fast path (gs_grid4.cu): every structure of the
    enumeration, grids of different lengths per model (including a single
    value), against the oracle walk over all configs."""
    rng = np.random.default_rng(n_rec + sum(glen))
    cert = rng.random((n_rec, 4))
    if ties:
        cert = np.round(cert, 1)
    corr = (rng.random((n_rec, 4)) < 0.6).astype(np.uint8)
    grids = []
    for j, g in enumerate(glen):
        q = np.quantile(cert[:, j], np.arange(1, g) / g) if g > 1 else []
        vals = sorted({0.0} | {float(x) for x in q})
        while len(vals) < g:  # ties collapsed quantiles: pad above the data
            vals.append(vals[-1] + 1.0)
        grids.append(np.array(vals[:g]))
    cost1 = rng.uniform(10, 500, 4)
    sw, (acc, cost, frac, nc) = _sweep(cert, corr, grids, cost1)
    sm, thr, ns = oracle.grid_configs(grids)
    want = oracle.evaluate_encoded(cert, corr, sm, thr, ns, cost1, n_threads=8)
    assert np.array_equal(acc, want[0])
    assert np.array_equal(cost, want[1])
    assert np.array_equal(frac, want[2])
    assert np.array_equal(nc / n_rec, want[0])
    # repeat build + eval on the same workspace
    sw.build()
    again = sw.evaluate()
    assert np.array_equal(again.accuracy.cpu().numpy(), want[0])
    assert np.array_equal(again.forward_frac.cpu().numpy(), want[2])


def test_four_models_past_packed_field_range():
    """n_rec >= 2^21 leaves the 21-bit packed fast path for the general
    path; sampled configs of every structure still match the oracle."""
    from paper_2406_14424_b200.gridsweep import GridSweep, structures
    rng = np.random.default_rng(21)
    n = (1 << 21) + 3
    cert = rng.random((n, 4))
    corr = (rng.random((n, 4)) < 0.7).astype(np.uint8)
    grids = [np.array(sorted({0.0} | set(np.quantile(cert[:, j], np.arange(1, 8) / 8).tolist())))
             for j in range(4)]
    cost1 = np.array([1.0, 4.0, 16.0, 64.0])
    sw = GridSweep(cert, corr, grids, cost1)
    res = sw.evaluate()
    pick = []
    for _, b, cnt in structures(4, sw.grid_len):
        pick.extend(sorted(set(rng.integers(b, b + cnt, size=min(cnt, 12)).tolist())))
    pick = np.array(pick)
    sm, thr, ns = oracle.grid_configs(grids)
    want = oracle.evaluate_encoded(cert, corr, sm[pick], thr[pick], ns[pick], cost1, n_threads=8)
    assert np.array_equal(res.accuracy.cpu().numpy()[pick], want[0])
    assert np.array_equal(res.mean_cost.cpu().numpy()[pick], want[1])
    assert np.array_equal(res.forward_frac.cpu().numpy()[pick], want[2])


@pytest.mark.parametrize("chunks", [1, 3, 8])
def test_streamed_build_equals_build(chunks):
    """gs_grid_accumulate over host slices (copies overlapped with binning)
    + gs_grid_finish gives the same tables as one gs_grid_build."""
    import torch
    from paper_2406_14424_b200.gridsweep import GridSweep
    rng = np.random.default_rng(chunks)
    cert, corr, grids, cost1 = _random_case(rng, 50_001, 4, 15)
    ref = GridSweep(cert, corr, grids, cost1).evaluate(n_correct=True)
    host_c = torch.from_numpy(cert).pin_memory()
    host_k = torch.from_numpy(corr).pin_memory()
    dev_c = torch.zeros(cert.shape, dtype=torch.float64, device="cuda")
    dev_k = torch.zeros(corr.shape, dtype=torch.uint8, device="cuda")
    sw = GridSweep(dev_c, dev_k, grids, cost1, build=False)
    assert sw.info.fast_path == 2  # one-shot builds take the bucket-sort kernels
    for _ in range(2):  # a second streamed build on the same workspace
        sw.build_streamed(host_c, host_k, chunks=chunks)
        got = sw.evaluate(n_correct=True)
        for a, b in ((got.accuracy, ref.accuracy), (got.mean_cost, ref.mean_cost),
                     (got.forward_frac, ref.forward_frac), (got.n_correct, ref.n_correct)):
            assert torch.equal(a, b)
    assert torch.equal(dev_c.cpu(), host_c)


def test_streamed_build_rejects_general_path():
    import torch
    from paper_2406_14424_b200.gridsweep import GridSweep
    rng = np.random.default_rng(3)
    cert, corr, grids, cost1 = _random_case(rng, 1000, 3, 5)
    sw = GridSweep(cert, corr, grids, cost1, build=False)
    assert sw.info.fast_path == 0
    with pytest.raises(ValueError):
        sw.build_streamed(torch.from_numpy(cert), torch.from_numpy(corr))


@pytest.mark.parametrize("glen", [(150, 40, 120, 10), (60, 300, 64, 5), (255, 3, 200, 2),
                                  (150, 3, 200, 2), (10, 150, 5), (40, 250, 3),
                                  (6, 1000, 9, 3), (6, 1500, 9, 3), (3, 14, 9, 3),
                                  (30, 30, 30, 30, 30)])
def test_four_model_large_uneven_grids(glen):
    """Grids near and past the fast path's shared-memory bounds (the plan
    falls back to the general path past them), and general-path slabs wide
    enough to be split across two CTAs (which must not re-zero the histogram
    in place: regression); sampled configs of every structure against the
    oracle walk."""
    from paper_2406_14424_b200.gridsweep import GridSweep, structures
    rng = np.random.default_rng(sum(glen))
    n = 40_000
    m = len(glen)
    cert = rng.random((n, m))
    corr = (rng.random((n, m)) < 0.6).astype(np.uint8)
    grids = [np.concatenate([[0.0], np.sort(rng.random(g - 1))]) for g in glen]
    cost1 = np.array([1.0, 3.0, 9.0, 27.0, 81.0])[:m]
    sw = GridSweep(cert, corr, grids, cost1)
    res = sw.evaluate(n_correct=True)
    pick = []
    for _, b, cnt in structures(m, sw.grid_len):
        pick.extend(sorted(set(rng.integers(b, b + cnt, size=min(cnt, 60)).tolist())))
    pick = np.array(pick)
    sm, thr, ns = (t.cpu().numpy() for t in sw.decode(pick))
    want = oracle.evaluate_encoded(cert, corr, sm, thr, ns, cost1, n_threads=8)
    assert np.array_equal(res.accuracy.cpu().numpy()[pick], want[0])
    assert np.array_equal(res.mean_cost.cpu().numpy()[pick], want[1])
    assert np.array_equal(res.forward_frac.cpu().numpy()[pick], want[2])
    assert np.array_equal(res.n_correct.cpu().numpy()[pick] / n, want[0])


def test_sweep_pipeline_fronts_equal_single_sweeps():
    """SweepPipeline (H2D of set i+1 overlapped with set i's sweep and front
    read-back) returns exactly the rows of one-at-a-time sweeps, in order."""
    import torch
    from paper_2406_14424_b200.gridsweep import GridSweep, front_host, pareto_counts
    from paper_2406_14424_b200.pipeline import SweepPipeline
    rng = np.random.default_rng(12)
    n, m = 30_000, 4
    grids = [np.concatenate([[0.0], np.sort(rng.random(19))]) for _ in range(m)]
    cost1 = np.array([1.0, 4.0, 16.0, 64.0])
    sets = []
    for _ in range(5):
        cert = rng.random((n, m))
        corr = (rng.random((n, m)) < 0.7).astype(np.uint8)
        sets.append((torch.from_numpy(cert).pin_memory(), torch.from_numpy(corr).pin_memory()))
    want = []
    for c, k in sets:
        sw = GridSweep(c.numpy(), k.numpy(), grids, cost1)
        res = sw.evaluate(n_correct=True)
        want.append(front_host(pareto_counts(res.n_correct, res.mean_cost, n), res).copy())
    pipe = SweepPipeline(n, m, grids, cost1)
    tickets = [pipe.submit(c, k) for c, k in sets]
    got = [pipe.result(t) for t in tickets]
    for a, b in zip(got, want):
        assert np.array_equal(a, b)
    pipe.drain()


def _equal_results(a, b):
    import torch
    for x, y in ((a.accuracy, b.accuracy), (a.mean_cost, b.mean_cost),
                 (a.forward_frac, b.forward_frac), (a.n_correct, b.n_correct)):
        assert torch.equal(x, y)


@pytest.mark.parametrize("skew", [False, True])
def test_sorted_build_matches_streamed_build(skew):
    """The bucket-sort build (gs_grid_build) and the histogram build
    (gs_grid_accumulate + gs_grid_finish) give identical tables, alternating
    on one workspace.  skew: 80% of the records share model 1's bin, so that
    bucket holds > 2^16 keys (the gather's wide counters)."""
    import torch
    from paper_2406_14424_b200.gridsweep import GridSweep
    rng = np.random.default_rng(17)
    n = 300_000 if skew else 60_000
    cert, corr, grids, cost1 = _random_case(rng, n, 4, 20)
    if skew:
        cert[: 4 * n // 5, 1] = 0.5
        q = np.quantile(cert[:, 1], np.arange(1, 20) / 20)
        grids[1] = np.array(sorted({0.0} | {float(x) for x in q}))
    sw = GridSweep(cert, corr, grids, cost1, build=False)
    assert sw.info.fast_path == 2
    host_c = torch.from_numpy(cert).pin_memory()
    host_k = torch.from_numpy(corr).pin_memory()
    sw.build()
    a = sw.evaluate(n_correct=True)
    sw.build_streamed(host_c, host_k, chunks=3)
    b = sw.evaluate(n_correct=True)
    _equal_results(a, b)
    sw.build()
    _equal_results(sw.evaluate(n_correct=True), b)
    # spot check against the oracle walk
    pick = np.sort(rng.choice(sw.n_configs, size=48, replace=False))
    sm, thr, ns = oracle.grid_configs(grids)
    want = oracle.evaluate_encoded(cert, corr, sm[pick], thr[pick], ns[pick], cost1, n_threads=8)
    assert np.array_equal(a.accuracy.cpu().numpy()[pick], want[0])
    assert np.array_equal(a.mean_cost.cpu().numpy()[pick], want[1])


def test_build_passes_split():
    """GS_GRID_BUILD_RECORDS_PASS then GS_GRID_BUILD_TABLES_PASS == one build."""
    from paper_2406_14424_b200.gridsweep import GridSweep
    rng = np.random.default_rng(5)
    cert, corr, grids, cost1 = _random_case(rng, 40_000, 4, 30)
    sw = GridSweep(cert, corr, grids, cost1)
    a = sw.evaluate(n_correct=True)
    sw.build(part="records")
    sw.build(part="tables")
    _equal_results(sw.evaluate(n_correct=True), a)


@pytest.mark.parametrize("n_rec", [5, 1025, 3 * 1024 + 7, 150_001])
def test_sorted_build_unaligned_inputs(n_rec):
    """The bucket-sort build reads records through a cp.async ring when the
    rows are 16-byte aligned and the correct words 4-byte aligned, else with
    scalar loads: views offset by 8 B (certainty) and 1 B (correct) take the
    second path and must give the same tables (and the oracle's values)."""
    import torch
    from paper_2406_14424_b200.gridsweep import GridSweep
    rng = np.random.default_rng(n_rec)
    cert, corr, grids, cost1 = _random_case(rng, n_rec, 4, 9)
    a = GridSweep(cert, corr, grids, cost1)
    assert a.info.fast_path == 2
    big_c = torch.empty(n_rec * 4 + 1, dtype=torch.float64, device="cuda")
    big_k = torch.empty(n_rec * 4 + 1, dtype=torch.uint8, device="cuda")
    vc = big_c[1:].view(n_rec, 4)
    vk = big_k[1:].view(n_rec, 4)
    vc.copy_(torch.from_numpy(cert))
    vk.copy_(torch.from_numpy(corr))
    assert vc.data_ptr() % 16 == 8 and vk.data_ptr() % 4 == 1
    b = GridSweep(vc, vk, grids, cost1)
    assert b.cert.data_ptr() == vc.data_ptr()
    _equal_results(a.evaluate(n_correct=True), b.evaluate(n_correct=True))
    if n_rec <= 5000:
        sm, thr, ns = oracle.grid_configs(grids)
        want = oracle.evaluate_encoded(cert, corr, sm, thr, ns, cost1, n_threads=8)
        assert np.array_equal(b.evaluate().accuracy.cpu().numpy(), want[0])


@pytest.mark.parametrize("n_rec,levels,ties", [(10_000, 100, False), (777, 12, True), (1, 3, False),
                                              (70_000, 20, True)])
def test_batched_three_model_sweeps_match_single(n_rec, levels, ties):
    """gs_grid_sweep_batched: each set's rows equal that set's own
    GridSweep (one launch for every set, a CTA per set; 16-bit packed
    counters below 2^16 records, 32-bit ones from there)."""
    from paper_2406_14424_b200.gridsweep import GridSweep, sweep_batched
    rng = np.random.default_rng(n_rec + levels)
    sets = [_random_case(rng, n_rec, 3, levels, ties) for _ in range(5)]
    # one grid-length triple for the batch: trim every set's grids to the shortest
    glen = [min(len(s[2][j]) for s in sets) for j in range(3)]
    grids = [[s[2][j][:glen[j]] for j in range(3)] for s in sets]
    cost1 = sets[0][3]
    cert = np.stack([s[0] for s in sets])
    corr = np.stack([s[1] for s in sets])
    res = sweep_batched(cert, corr, grids, cost1)
    for i in range(len(sets)):
        ref = GridSweep(cert[i], corr[i], grids[i], cost1).evaluate()
        assert torch_equal(res.accuracy[i], ref.accuracy)
        assert torch_equal(res.mean_cost[i], ref.mean_cost)
        assert torch_equal(res.forward_frac[i], ref.forward_frac)


def torch_equal(a, b):
    import torch
    return bool(torch.equal(a, b))


def test_batched_sweep_config1_golden():
    """Set 0 of a batch is config 1 (the reference's golden values)."""
    from paper_2406_14424_b200 import synth
    from paper_2406_14424_b200.gridsweep import sweep_batched
    g = golden("config1.npz")
    cert0, corr0 = synth.validation_matrices(3, 10_000, 0.8, 0)
    cert1, corr1 = synth.validation_matrices(3, 10_000, 0.8, 1)
    grids = [g["grid0"], g["grid1"], g["grid2"]]
    res = sweep_batched(np.stack([cert0, cert1]), np.stack([corr0, corr1]), [grids, grids],
                        g["cost1"])
    assert np.array_equal(res.accuracy[0].cpu().numpy(), g["acc"])
    assert np.array_equal(res.mean_cost[0].cpu().numpy(), g["cost"])
    assert np.array_equal(res.forward_frac[0].cpu().numpy(), g["frac"])


def test_sorted_build_near_record_limit():
    """2M records (just under the packed fields' 2^21): the sort's record
    ranges no longer leave room for the cp.async ring, so the register path
    runs; tables equal the histogram build's."""
    import torch
    from paper_2406_14424_b200.gridsweep import GridSweep
    rng = np.random.default_rng(21)
    n = 2_000_000
    cert, corr, grids, cost1 = _random_case(rng, n, 4, 20)
    sw = GridSweep(cert, corr, grids, cost1, build=False)
    assert sw.info.fast_path == 2
    sw.build()
    a = sw.evaluate(n_correct=True)
    sw.build_streamed(torch.from_numpy(cert).pin_memory(), torch.from_numpy(corr).pin_memory(),
                      chunks=2)
    _equal_results(sw.evaluate(n_correct=True), a)
    pick = np.sort(rng.choice(sw.n_configs, size=12, replace=False))
    sm, thr, ns = oracle.grid_configs(grids)
    want = oracle.evaluate_encoded(cert, corr, sm[pick], thr[pick], ns[pick], cost1, n_threads=8)
    assert np.array_equal(a.accuracy.cpu().numpy()[pick], want[0])


def test_batched_sweep_rejects_bad_input():
    from paper_2406_14424_b200.gridsweep import BatchedSweep
    rng = np.random.default_rng(2)
    cert = rng.random((2, 50, 3))
    corr = (rng.random((2, 50, 3)) < 0.5).astype(np.uint8)
    g = [np.array([0.0, 0.5]), np.array([0.0, 0.3, 0.6]), np.array([0.0])]
    cost1 = [1.0, 2.0, 3.0]
    with pytest.raises(ValueError):  # one grid triple for two sets
        BatchedSweep(cert, corr, [g], cost1)
    with pytest.raises(ValueError):  # lengths differ between sets
        BatchedSweep(cert, corr, [g, [g[0], g[1][:2], g[2]]], cost1)
    with pytest.raises(ValueError):  # not increasing
        BatchedSweep(cert, corr, [g, [g[0][::-1], g[1], g[2]]], cost1)
    with pytest.raises(ValueError):  # a grid per model
        BatchedSweep(rng.random((2, 50, 4)), np.zeros((2, 50, 4), np.uint8), [g, g], cost1)
    res = BatchedSweep(cert, corr, [g, g], cost1).run()
    assert tuple(res.accuracy.shape) == (2, 3 + 2 * 2 + 3 + 2 * 3)


@pytest.mark.parametrize("n_rec,glen,ties", [
    (3000, (7, 5, 9, 11, 3), False), (5000, (12, 1, 6, 20, 4), True), (1, (1, 1, 1, 1, 1), False),
    (80_000, (2, 3, 2, 4, 2), True)])
def test_five_model_slab_walk_vs_oracle(n_rec, glen, ties):
    """The five-model path (gs_sweep5.cu: slab-sorted build, b0 walk, faces
    for the regular eval) over uneven grids, heavy ties, a b0 slab past 2^16
    records (the 21-bit variant of the slab pass), every config vs the
    oracle walk."""
    rng = np.random.default_rng(n_rec + sum(glen))
    cert = np.round(rng.random((n_rec, 5)), 1) if ties else rng.random((n_rec, 5))
    corr = (rng.random((n_rec, 5)) < 0.6).astype(np.uint8)
    grids = [np.concatenate([[0.0], np.sort(rng.choice(np.unique(cert[:, j]),
                                                       size=min(g - 1, len(np.unique(cert[:, j]))),
                                                       replace=False))])
             if g > 1 else np.array([0.0]) for j, g in enumerate(glen)]
    grids = [np.unique(g) for g in grids]
    cost1 = rng.uniform(100, 5000, 5)
    sw, (acc, cost, frac, nc) = _sweep(cert, corr, grids, cost1)
    assert sw.info.build_launches == 5, "the five-model slab path did not run"
    sm, thr, ns = oracle.grid_configs(grids)
    want = oracle.evaluate_encoded(cert, corr, sm, thr, ns, cost1, n_threads=8)
    assert np.array_equal(acc, want[0])
    assert np.array_equal(cost, want[1])
    assert np.array_equal(frac, want[2])
    idx, _ = sw.pareto()
    assert np.array_equal(idx.cpu().numpy(), np.flatnonzero(oracle.pareto_keep(want[0], want[1])))


def test_config4b_shape_sampled_vs_oracle():
    """Config 4b (5 models, 100-level grids, 100k records, C = 105,101,005):
    the slab path, configs of every structure sampled against the oracle."""
    from paper_2406_14424_b200 import synth
    from paper_2406_14424_b200.cascades import grid_values
    from paper_2406_14424_b200.gridsweep import GridSweep, structures
    cert, corr = synth.validation_matrices(5, 100_000, 0.8, 5)
    grids = [np.array(grid_values(cert[:, j], 100)) for j in range(5)]
    cost1 = np.array([1.0, 4.0, 16.0, 64.0, 256.0])
    sw = GridSweep(cert, corr, grids, cost1)
    assert sw.n_configs == 105_101_005 and sw.info.build_launches == 5
    res = sw.evaluate()
    rng = np.random.default_rng(1)
    pick = []
    for _, b, n in structures(5, sw.grid_len):
        pick.extend(sorted(set(rng.integers(b, b + n, size=min(n, 24)).tolist())))
    pick = np.array(pick)
    sm, thr, ns = (t.cpu().numpy() for t in sw.decode(pick))
    want = oracle.evaluate_encoded(cert, corr, sm, thr, ns, cost1, n_threads=8)
    import torch
    ip = torch.from_numpy(pick).cuda()
    assert np.array_equal(res.accuracy[ip].cpu().numpy(), want[0])
    assert np.array_equal(res.mean_cost[ip].cpu().numpy(), want[1])
    assert np.array_equal(res.forward_frac[ip].cpu().numpy(), want[2])


def _sweep_general(cert, corr, grids, cost1):
    """The same sweep through the general path (GS_GRID_GENERAL=1 at plan time)."""
    os.environ["GS_GRID_GENERAL"] = "1"
    try:
        from paper_2406_14424_b200.gridsweep import GridSweep
        sw = GridSweep(cert, corr, grids, cost1)
        assert sw.info.fast_path == 0 and sw.info.build_launches != 5
        return sw, sw.evaluate()
    finally:
        del os.environ["GS_GRID_GENERAL"]


def test_config4b_full_product_vs_general_path():
    """Config 4b over its whole enumeration (105,101,005 configs): the
    five-model slab path (narrow and wide T slabs, faces, regular eval) equals
    the general path (dense histogram, in-place prefixes, general eval) bit
    for bit on every output; every 50,000th config also against the oracle."""
    import torch
    from paper_2406_14424_b200 import synth
    from paper_2406_14424_b200.cascades import grid_values
    from paper_2406_14424_b200.gridsweep import GridSweep
    cert, corr = synth.validation_matrices(5, 100_000, 0.8, 5)
    grids = [np.array(grid_values(cert[:, j], 100)) for j in range(5)]
    cost1 = np.array([1.0, 4.0, 16.0, 64.0, 256.0])
    sw = GridSweep(cert, corr, grids, cost1)
    assert sw.n_configs == 105_101_005 and sw.info.build_launches == 5
    fast = sw.evaluate()
    gen_sw, gen = _sweep_general(cert, corr, grids, cost1)
    assert gen_sw.n_configs == sw.n_configs
    for a, b in ((fast.accuracy, gen.accuracy), (fast.mean_cost, gen.mean_cost),
                 (fast.forward_frac, gen.forward_frac)):
        assert torch.equal(a.view(torch.int64), b.view(torch.int64))
    pick = np.arange(0, sw.n_configs, 50_000)
    sm, thr, ns = (t.cpu().numpy() for t in sw.decode(pick))
    want = oracle.evaluate_encoded(cert, corr, sm, thr, ns, cost1, n_threads=os.cpu_count() or 8)
    ip = torch.from_numpy(pick).cuda()
    assert np.array_equal(fast.accuracy[ip].cpu().numpy(), want[0])
    assert np.array_equal(fast.mean_cost[ip].cpu().numpy(), want[1])
    assert np.array_equal(fast.forward_frac[ip].cpu().numpy(), want[2])


@pytest.mark.parametrize("n_rec,M,glen", [(2**24 + 1001, 3, (4, 3, 2)), (2**26 + 3, 2, (3, 2))])
def test_general_path_past_f32_and_rcp_ranges(n_rec, M, glen):
    """Record sets past 2^24 (the f32 fallback histogram would round: the
    16-bit packed table overflows and the fallback counts in u32) and past
    2^26 (the three-op division's range: IEEE division instead), every config
    vs the oracle."""
    rng = np.random.default_rng(n_rec)
    cert = rng.random((n_rec, M))
    corr = (rng.random((n_rec, M)) < 0.7).astype(np.uint8)
    grids = [np.sort(rng.random(g)) for g in glen]
    cost1 = np.arange(1.0, M + 1.0) * 3.0
    sw, (acc, cost, frac, nc) = _sweep(cert, corr, grids, cost1)
    assert sw.info.fast_path == 0
    sm, thr, ns = oracle.grid_configs(grids)
    want = oracle.evaluate_encoded(cert, corr, sm, thr, ns, cost1, n_threads=os.cpu_count() or 8)
    assert np.array_equal(acc, want[0])
    assert np.array_equal(cost, want[1])
    assert np.array_equal(frac, want[2])


@pytest.mark.parametrize("M", [2, 4, 5])
def test_batched_sweep_other_model_counts(M):
    """Sets of 2, 4 or 5 models: the batched API runs each set's sweep (no
    single-launch kernel for them) and every row equals that set's GridSweep."""
    from paper_2406_14424_b200.gridsweep import BatchedSweep, GridSweep
    rng = np.random.default_rng(M)
    R, n = 3, 2000
    cert = rng.random((R, n, M))
    corr = (rng.random((R, n, M)) < 0.6).astype(np.uint8)
    lens = [5, 4, 6, 3, 2][:M]
    grids = [[np.sort(rng.choice(cert[s, :, j], size=lens[j], replace=False)) for j in range(M)]
             for s in range(R)]
    cost1 = np.arange(1.0, M + 1.0) * 2.0
    res = BatchedSweep(cert, corr, grids, cost1).run()
    for s in range(R):
        one = GridSweep(cert[s], corr[s], grids[s], cost1).evaluate()
        assert np.array_equal(res.accuracy[s].cpu().numpy(), one.accuracy.cpu().numpy())
        assert np.array_equal(res.mean_cost[s].cpu().numpy(), one.mean_cost.cpu().numpy())
        assert np.array_equal(res.forward_frac[s].cpu().numpy(), one.forward_frac.cpu().numpy())
