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
