"""The reference-facing cascade API (paper_2406_14424_b200.cascades) on the
GPU, checked like the reference's own test_cascades.py / acceptance C1."""

import numpy as np
import pytest

import golden_inputs as gi
from conftest import golden
from oracle import oracle

pytestmark = pytest.mark.gpu


def _profiles2():
    from paper_2406_14424_b200.types import ModelProfile, ProfileSet
    return ProfileSet([ModelProfile("small", 4_000_000_000, {1: 5_000, 2: 8_000, 4: 12_000}),
                       ModelProfile("large", 10_000_000_000, {1: 20_000, 2: 32_000, 4: 48_000})])


def _record(sid, small_cert, small_ok, large_cert, large_ok):
    from paper_2406_14424_b200.types import ModelOutput, ValidationRecord
    return ValidationRecord(sample_id=sid, outputs={
        "small": ModelOutput(scores=(0.5 + small_cert / 2, 0.5 - small_cert / 2), correct=small_ok),
        "large": ModelOutput(scores=(0.5 + large_cert / 2, 0.5 - large_cert / 2), correct=large_ok)})


def test_evaluate_cascade_by_hand():
    from paper_2406_14424_b200.cascades import evaluate_cascade
    from paper_2406_14424_b200.types import Cascade, ValidationSet
    v = ValidationSet(records=(_record(0, 0.8, True, 0.9, True), _record(1, 0.6, False, 0.9, True),
                               _record(2, 0.4, True, 0.9, False), _record(3, 0.2, False, 0.9, True)))
    ev = evaluate_cascade(Cascade(("small", "large"), (0.5,)), v, _profiles2())
    assert ev.accuracy == pytest.approx(0.5)
    assert ev.forward_fraction == {"small": 1.0, "large": 0.5}
    assert ev.mean_cost == pytest.approx(15_000.0)
    with pytest.raises(ValueError):
        evaluate_cascade(Cascade(("ghost",), ()), v, _profiles2())


def test_c1_through_records():
    """Acceptance C1: ragged Python score tuples -> device matrices ->
    evaluate_cascades, equal (==) to the reference's outputs."""
    from paper_2406_14424_b200 import cascades
    from paper_2406_14424_b200.types import (Cascade, ModelOutput, ModelProfile, ProfileSet,
                                             ValidationRecord, ValidationSet)
    g = golden("c1.npz")
    for i, fx in enumerate(gi.c1_fixtures()[:40]):
        M = len(fx["mids"])
        profiles = ProfileSet([ModelProfile(m, 1_000_000, {1: c})
                               for m, c in zip(fx["mids"], fx["cost1"])])
        recs = [ValidationRecord(sample_id=r, outputs={
            m: ModelOutput(scores=tuple(float(x) for x in fx["scores"][r * M + j, :fx["lens"][r * M + j]]),
                           correct=bool(fx["correct"][r, j])) for j, m in enumerate(fx["mids"])})
            for r in range(fx["n_rec"])]
        val = ValidationSet(recs)
        cert, corr = cascades.matrices(val, profiles)
        assert np.array_equal(cert, g[f"f{i}_cert"]) and np.array_equal(corr, g[f"f{i}_corr"])
        cascs = [Cascade(stages=s, thresholds=t) for s, t in fx["cascades"]]
        evs = cascades.evaluate_cascades(cascs, val, profiles)
        assert [e.accuracy for e in evs] == list(g[f"f{i}_acc"])
        assert [e.mean_cost for e in evs] == list(g[f"f{i}_cost"])


def test_pareto_filter_matches_reference():
    from paper_2406_14424_b200.cascades import CascadeEval, pareto_filter
    from paper_2406_14424_b200.types import Cascade
    g = golden("pareto.npz")
    for t, (acc, cost) in enumerate(gi.pareto_cases()):
        items = [(Cascade((f"m{i}",), ()), CascadeEval(float(a), float(c), {}))
                 for i, (a, c) in enumerate(zip(acc, cost))]
        kept = pareto_filter(items)
        want = [items[i] for i in np.flatnonzero(g[f"p{t}_keep"])]
        assert kept == want
    assert pareto_filter([]) == []


def test_sweep_grid_front_is_exact():
    from paper_2406_14424_b200 import cascades, synth
    p = synth.make_profiles()
    v = synth.make_validation_arrays(p, n_samples=4000, seed=2)
    grid = cascades.build_threshold_grid(v, p, levels=20)
    front = cascades.sweep_grid(v, p, grid)
    cert, corr = cascades.matrices(v, p)
    grids = [np.array(grid.per_model[m]) for m in p.model_ids]
    sm, thr, ns = oracle.grid_configs(grids)
    acc, cost, frac = oracle.evaluate_encoded(cert, corr, sm, thr, ns, p.cost1())
    keep = np.flatnonzero(oracle.pareto_keep(acc, cost))
    assert np.array_equal(front.config_index, keep)
    assert [e.accuracy for e in front.evals] == list(acc[keep])
    assert [e.mean_cost for e in front.evals] == list(cost[keep])
    # the decoded cascades score the same through the list path
    evs = cascades.evaluate_cascades(front.cascades, v, p)
    assert [e.accuracy for e in evs] == list(acc[keep])


def test_jsonl_ingest_feeds_the_same_matrices(tmp_path):
    """formats.load_validation_arrays (native reader + device certainty) gives
    bit-identical matrices to the record path, and a sweep over them equals
    the oracle walk."""
    from paper_2406_14424_b200 import formats, synth
    from paper_2406_14424_b200.cascades import matrices
    from paper_2406_14424_b200.types import ModelOutput, ValidationRecord, ValidationSet
    profiles = synth.make_profiles(n_models=3)
    va = synth.binary_logit_arrays(profiles, 3000, 0.8, seed=4, dtype=np.float64)
    vs = ValidationSet([ValidationRecord(
        sample_id=i, outputs={m: ModelOutput(scores=tuple(float(x) for x in va.scores[m][i]),
                                             correct=bool(va.correct[i, j]))
                              for j, m in enumerate(profiles.model_ids)})
        for i in range(3000)])
    path = tmp_path / "v.jsonl"
    formats.save_validation(vs, path)
    arr = formats.load_validation_arrays(path)
    c_ref, k_ref = matrices(vs, profiles)
    c_arr, k_arr = matrices(arr, profiles)
    assert np.array_equal(c_ref, c_arr) and np.array_equal(k_ref, k_arr)
    col = tmp_path / "v.gsvc"
    formats.save_validation_columnar(arr, col)
    c_col, k_col = matrices(formats.load_validation_columnar(col), profiles)
    assert np.array_equal(c_ref, c_col) and np.array_equal(k_ref, k_col)
