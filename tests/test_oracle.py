"""The oracle (oracle/) pinned against golden vectors captured from the
reference (tests/golden/make_golden.py).  CPU only."""

import hashlib
import json

import numpy as np
import pytest

import golden_inputs as gi
from conftest import golden
from oracle import oracle


def _sha(*arrays) -> bytes:
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return h.digest()


def test_random_problems_match_reference_numba():
    g = golden("kernels.npz")
    rng = np.random.default_rng(12345)
    for t in range(5):
        args = gi.random_problem(rng)
        assert _sha(*args) == g[f"rp{t}_sha"].tobytes(), "input generator drifted"
        acc, cost, frac = oracle.evaluate_encoded(*args)
        assert np.array_equal(acc, g[f"rp{t}_acc"])
        assert np.array_equal(cost, g[f"rp{t}_cost"])
        assert np.array_equal(frac, g[f"rp{t}_frac"])


def test_bench_problem_matches_reference_numba():
    g = golden("kernels.npz")
    args = gi.bench_problem(4000, 6, 200, 0)
    assert _sha(*args) == g["bench_sha"].tobytes()
    for threads in (1, 4):
        acc, cost, frac = oracle.evaluate_encoded(*args, n_threads=threads)
        assert np.array_equal(acc, g["bench_acc"])
        assert np.array_equal(cost, g["bench_cost"])
        assert np.array_equal(frac, g["bench_frac"])


def test_python_walk_pins_c_port(rng):
    for _ in range(3):
        args = gi.random_problem(rng, n_rec=60, n_models=5, n_casc=25, max_len=5)
        a = oracle.evaluate_encoded(*args)
        b = oracle.walk_python(*args)
        for x, y in zip(a, b):
            assert np.array_equal(x, y)


def test_c1_fixtures_certainty_and_walk():
    g = golden("c1.npz")
    for i, fx in enumerate(gi.c1_fixtures()):
        cert = oracle.margin_rows(fx["scores"], fx["lens"]).reshape(fx["n_rec"], len(fx["mids"]))
        assert np.array_equal(cert, g[f"f{i}_cert"])
        assert np.array_equal(fx["correct"], g[f"f{i}_corr"])
        sm, thr, ns = gi.encode(fx["cascades"], fx["mids"])
        acc, cost, frac = oracle.evaluate_encoded(cert, fx["correct"], sm, thr, ns,
                                                  np.asarray(fx["cost1"], dtype=np.float64))
        assert np.array_equal(acc, g[f"f{i}_acc"])
        assert np.array_equal(cost, g[f"f{i}_cost"])
        assert np.array_equal(frac, g[f"f{i}_frac"])


def test_config1_full_grid_matches_reference():
    from paper_2406_14424_b200 import synth
    g = golden("config1.npz")
    cert, corr = synth.validation_matrices(3, 10_000, 0.8, 0)
    assert _sha(cert, corr) == g["cert_sha"].tobytes()
    grids = [g["grid0"], g["grid1"], g["grid2"]]
    sm, thr, ns = oracle.grid_configs(grids)
    assert sm.shape[0] == 10_303 == oracle.grid_n_configs([len(x) for x in grids])
    py = gi.grid_configs_py(grids)
    assert all(np.array_equal(a, b) for a, b in zip((sm, thr, ns), py))
    acc, cost, frac = oracle.evaluate_encoded(cert, corr, sm, thr, ns, g["cost1"], n_threads=8)
    assert np.array_equal(acc, g["acc"])
    assert np.array_equal(cost, g["cost"])
    assert np.array_equal(frac, g["frac"])


def test_certainty_restatements():
    g = golden("certainty.npz")
    rows, lens = gi.certainty_tuples()
    ref = g["tuples"]
    got = np.array([oracle.certainty(tuple(rows[i, : lens[i]])) for i in range(rows.shape[0])])
    assert np.array_equal(got, ref)
    assert np.array_equal(oracle.margin_rows(rows, lens), ref)
    logits = gi.logits_f32(seed=3, n=256, n_cls=1000)
    assert _sha(logits) == g["logits_sha"].tobytes()
    assert np.array_equal(oracle.margin_rows(logits), g["logits"])
    with pytest.raises(ValueError):
        oracle.certainty(())


def test_pareto_restatements():
    g = golden("pareto.npz")
    for t, (acc, cost) in enumerate(gi.pareto_cases()):
        want = g[f"p{t}_keep"]
        assert np.array_equal(oracle.pareto_keep(acc, cost), want)
        assert np.array_equal(oracle.pareto_keep_quadratic(acc, cost), want)


def test_finish_batch_restatement():
    g = golden("engine.npz")
    for t, case in enumerate(gi.engine_cases()):
        want = json.loads(str(g[f"e{t}"]))
        replicas = case["replicas"]
        gears = []
        for gd in case["gears"]:
            mids = case["mids"]
            rep_idx, cum = [], []
            for m in gd["stages"]:
                idxs = [i for i, (rid, mm, _) in enumerate(replicas) if mm == m]
                w = np.array([gd["weights"][m][replicas[i][0]] for i in idxs])
                rep_idx.append(np.array(idxs))
                cum.append(np.cumsum(w))
            gears.append(dict(stage_model=[mids.index(m) for m in gd["stages"]],
                              thresholds=list(gd["thresholds"]) + [None],
                              replica_idx=rep_idx, cum_weights=cum))
        rng = np.random.default_rng(case["seed"])
        done, fwd = oracle.finish_batch(case["items"], gears, case["cert"], case["corr"], rng,
                                        case["now"])
        assert [list(d) for d in done] == [[a, int(b), c, d] for a, b, c, d in
                                          [tuple(x) for x in want["done"]]]
        queues = [[] for _ in replicas]
        for pos, r in fwd:
            it = case["items"][pos]
            queues[r].append([it["request_id"], it["stage"] + 1])
        assert queues == want["queues"]
        assert float(rng.random()) == want["rng_next"]


def test_extension_certainties_are_sane():
    x = gi.logits_f32(seed=4, n=64, n_cls=10)
    ms = oracle.max_softmax_rows(x)
    ent = oracle.entropy_rows(x)
    assert np.all((ms > 0) & (ms <= 1))
    assert np.all((ent >= -1e-12) & (ent <= 1 + 1e-12))
    flat = np.zeros((2, 10))
    assert np.allclose(oracle.entropy_rows(flat), 0.0)
    assert np.allclose(oracle.max_softmax_rows(flat), 0.1)
