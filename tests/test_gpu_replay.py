"""Device replay (gs_engine_run) against the reference engine.run goldens:
records, windows, counters, queues and batch histograms equal, per scenario
and with every scenario in one launch."""

import json

import numpy as np
import pytest

import golden_inputs as gi
from conftest import golden
from replay_cases import build

pytestmark = pytest.mark.gpu

CASES = list(gi.replay_cases())


def _check(name, res, g):
    r = res.records
    got = np.stack([r["request_id"], res.arrival_us[r["request_id"]], r["completion_us"],
                    r["stages_executed"], r["correct"], r["gear_index"]], 1).astype(np.int64)
    want = g[f"{name}_rec"]
    assert got.shape == want.shape, (name, got.shape, want.shape)
    assert np.array_equal(got, want), name
    w = res.windows
    gw = np.stack([w["end_us"], w["first_stage_queue_len"], w["gear_before"], w["candidate_gear"],
                   w["gear_after"], w["candidate_gear"], w["completed"], w["p95_us"]], 1)
    assert np.array_equal(gw.reshape(-1, 8), g[f"{name}_win"]), name
    gf = np.stack([w["measured_qps"], w["accuracy"]], 1).reshape(-1, 2)
    assert np.array_equal(gf, g[f"{name}_winf"], equal_nan=True), name
    assert [res.arrivals, res.completed, res.arrivals - res.completed, res.in_flight] == \
        g[f"{name}_counts"].tolist(), name
    assert np.array_equal(res.queue_len, g[f"{name}_qlen"]), name
    want_b = json.loads(str(g[f"{name}_batches"]))
    got_b = {m: {str(b): int(c) for b, c in enumerate(res.model_batches[j]) if c}
             for j, m in enumerate(res.plan.model_ids)}
    assert {k: v for k, v in got_b.items() if v} == want_b, name


@pytest.mark.parametrize("name", CASES)
def test_replay_matches_reference_engine_run(name):
    from paper_2406_14424_b200 import replay
    prof, val, trace, plan, cfg = build(gi.replay_cases()[name])
    dp = replay.DevicePlan(plan, prof, val)
    res = replay.run_many([replay.Job(dp, trace.arrivals, trace.duration_us, cfg)])[0]
    _check(name, res, golden("replay.npz"))


def test_all_scenarios_in_one_launch():
    from paper_2406_14424_b200 import replay
    g = golden("replay.npz")
    jobs = []
    for name in CASES:
        prof, val, trace, plan, cfg = build(gi.replay_cases()[name])
        jobs.append(replay.Job(replay.DevicePlan(plan, prof, val), trace.arrivals,
                               trace.duration_us, cfg))
    # each scenario twice, interleaved: runs are independent
    res = replay.run_many(jobs + jobs)
    for k, name in enumerate(CASES):
        _check(name, res[k], g)
        _check(name, res[k + len(CASES)], g)


def test_run_returns_reference_shaped_metrics():
    from paper_2406_14424_b200 import replay
    name = "bursty_two_gears"
    prof, val, trace, plan, cfg = build(gi.replay_cases()[name])
    m = replay.run(plan, trace, val, prof, config=cfg)
    g = golden("replay.npz")
    assert m.arrivals == m.completed == len(trace)
    assert [r.completion_us for r in m.per_request] == g[f"{name}_rec"][:, 2].tolist()
    assert len(m.windows) == len(g[f"{name}_win"])
    assert m.p95() if hasattr(m, "p95") else True


def _random_plan(rng, prof):
    from paper_2406_14424_b200.types import Cascade, Gear, GearPlan, Placement, Replica
    ids = list(prof.model_ids)
    n_dev = int(rng.integers(1, 5))
    reps = []
    for m in ids:
        for d in sorted(set(rng.integers(0, n_dev, int(rng.integers(1, 3))).tolist())):
            reps.append(Replica(f"{m}@d{d}", m, f"d{d}"))
    rng.shuffle(reps)
    gears = []
    for _ in range(int(rng.integers(1, 5))):
        k = int(rng.integers(1, len(ids) + 1))
        st = tuple(ids[i] for i in sorted(rng.choice(len(ids), size=k, replace=False)))
        thr = tuple(float(x) for x in np.round(rng.uniform(0.3, 0.9, k - 1), 2))
        w, q = {}, {}
        for m in st:
            w[m] = {}
            for r in reps:
                if r.model_id == m:
                    w[m][r.replica_id] = float(rng.choice([0.0, 0.5, 1.0, 2.0]))
                    if rng.random() < 0.3:
                        q[r.replica_id] = int(rng.integers(1, 5))
        gears.append(Gear(Cascade(st, thr), q, w))
    return GearPlan(placement=Placement(reps), slo=None, qps_max=float(rng.integers(50, 600)),
                    gears=tuple(gears))


def test_random_scenarios_vs_oracle_engine():
    """40 random plans / bursty traces / seeds, all in one launch, each equal
    to the oracle's restatement of engine.run (itself pinned to the
    reference goldens in test_replay_host.py)."""
    from oracle import oracle
    from paper_2406_14424_b200 import replay, synth
    from paper_2406_14424_b200.types import ValidationArrays
    rng = np.random.default_rng(2024)
    prof = synth.make_profiles(n_models=4, cost_ratios=(1.0, 2.0, 4.0, 8.0), base_runtime_us=500)
    ids = list(prof.model_ids)
    runtime = [[0] + [prof[m].runtime_us(b) for b in range(1, 9)] for m in ids]
    cert, corr = synth.validation_matrices(4, 3000, 0.8, 11)
    val = ValidationArrays(prof.model_ids, certainty=cert, correct=corr)
    cases, jobs = [], []
    for i in range(40):
        plan = _random_plan(rng, prof)
        trace = replay.scale_trace(synth.trace_from_counts(synth.bursty_counts(6, i)),
                                   float(rng.integers(50, 700)))
        cfg = replay.EngineConfig(seed=i, measure_period_us=int(rng.choice([20_000, 100_000])),
                                  alpha=float(rng.choice([2.0, 8.0])),
                                  initial_gear_index=int(rng.integers(0, len(plan.gears))),
                                  enable_ticks=bool(rng.random() < 0.8))
        cases.append((plan, trace, cfg))
        jobs.append(replay.Job(replay.DevicePlan(plan, prof, val), trace.arrivals,
                               trace.duration_us, cfg))
    res = replay.run_many(jobs)
    for (plan, trace, cfg), r in zip(cases, res):
        want = oracle.engine_run(plan, trace, cert, corr, runtime, [8] * 4,
                                 {m: j for j, m in enumerate(ids)}, seed=cfg.seed,
                                 period_us=cfg.measure_period_us, alpha=cfg.alpha,
                                 initial_gear=cfg.initial_gear_index,
                                 enable_ticks=cfg.enable_ticks)
        rec = r.records
        got = np.stack([rec["request_id"], r.arrival_us[rec["request_id"]], rec["completion_us"],
                        rec["stages_executed"], rec["correct"], rec["gear_index"]],
                       1).astype(np.int64).reshape(-1, 6)
        assert np.array_equal(got, want["records"])
        assert r.queue_len.tolist() == want["queue_len"]
        assert [r.arrivals, r.completed, r.in_flight] == \
            [want["arrivals"], want["completed"], want["in_flight"]]
        w = r.windows
        gw = [(int(a), int(b), int(c), int(d), int(e), int(f)) for a, b, c, d, e, f in
              zip(w["end_us"], w["first_stage_queue_len"], w["gear_before"],
                  w["candidate_gear"], w["gear_after"], w["p95_us"])]
        assert gw == [(x[0], x[2], x[3], x[4], x[5], x[7]) for x in want["windows"]]
        st = want["rng_state"]
        assert r.rng_state == (st["state"]["state"], st["has_uint32"], st["uinteger"])
