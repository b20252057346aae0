"""Deterministic input generators shared by tests/golden/make_golden.py (run
against the reference) and the tests (run against the oracle and the GPU).

Each generator restates how the reference's own tests build their inputs so
the golden outputs can be matched without storing large input arrays:
  random_problem  pkg/tests/test_kernels.py:7-19
  bench_problem   pkg/benchmarks/bench_kernels.py:25-49
  c1_fixtures     pkg/tests/test_acceptance.py:115-141
"""

from __future__ import annotations

import itertools

import numpy as np


def random_problem(rng, n_rec=200, n_models=4, n_casc=30, max_len=4):
    certainty = rng.random((n_rec, n_models))
    correct = (rng.random((n_rec, n_models)) < 0.7).astype(np.uint8)
    stage_model = np.full((n_casc, max_len), -1, dtype=np.int32)
    thresholds = np.zeros((n_casc, max_len))
    n_stages = np.zeros(n_casc, dtype=np.int32)
    for c in range(n_casc):
        k = int(rng.integers(1, max_len + 1))
        n_stages[c] = k
        stage_model[c, :k] = rng.choice(n_models, size=k, replace=False)
        thresholds[c, :k - 1] = rng.random(k - 1)
    cost1 = rng.uniform(1_000, 50_000, n_models)
    return certainty, correct, stage_model, thresholds, n_stages, cost1


def bench_problem(n_records, n_models, n_cascades, seed):
    rng = np.random.default_rng(seed)
    mids = [f"m{j}" for j in range(n_models)]
    cost1 = np.array([int(rng.integers(1_000, 60_000)) for _ in mids], dtype=np.float64)
    index = {m: j for j, m in enumerate(mids)}
    stages_list, thr_list = [], []
    for _ in range(n_cascades):
        k = int(rng.integers(1, n_models + 1))
        stages = tuple(rng.permutation(mids)[:k])
        stages_list.append(stages)
        thr_list.append(tuple(float(x) for x in rng.random(k - 1)))
    max_len = max(len(s) for s in stages_list)
    stage_model = np.full((n_cascades, max_len), -1, dtype=np.int32)
    thresholds = np.zeros((n_cascades, max_len))
    n_stages = np.zeros(n_cascades, dtype=np.int32)
    for ci, (s, t) in enumerate(zip(stages_list, thr_list)):
        n_stages[ci] = len(s)
        stage_model[ci, : len(s)] = [index[m] for m in s]
        thresholds[ci, : len(t)] = t
    certainty = rng.random((n_records, n_models))
    correct = (rng.random((n_records, n_models)) < 0.7).astype(np.uint8)
    return certainty, correct, stage_model, thresholds, n_stages, cost1


def c1_fixtures():
    """The 100 C1 fixtures with default_rng(7); ragged scores padded."""
    rng = np.random.default_rng(7)
    out = []
    for _ in range(100):
        n_models = int(rng.integers(1, 6))
        n_rec = int(rng.integers(1, 201))
        mids = [f"m{j}" for j in range(n_models)]
        cost1 = [int(rng.integers(500, 50_000)) for _ in mids]
        scores = np.zeros((n_rec * n_models, 4))
        lens = np.zeros(n_rec * n_models, dtype=np.int32)
        correct = np.zeros((n_rec, n_models), dtype=np.uint8)
        for i in range(n_rec):
            for j, _ in enumerate(mids):
                k = int(rng.integers(1, 5))
                s = rng.random(k)
                scores[i * n_models + j, :k] = s
                lens[i * n_models + j] = k
                correct[i, j] = 1 if rng.random() < 0.6 else 0
        cascs = []
        for _ in range(3):
            k = int(rng.integers(1, n_models + 1))
            stages = tuple(str(m) for m in rng.permutation(mids)[:k])
            cascs.append((stages, tuple(float(x) for x in rng.random(k - 1))))
        out.append(dict(mids=mids, cost1=cost1, n_rec=n_rec, scores=scores, lens=lens,
                        correct=correct, cascades=cascs))
    return out


def encode(cascs, mids):
    index = {m: j for j, m in enumerate(mids)}
    width = max(len(s) for s, _ in cascs)
    sm = np.full((len(cascs), width), -1, dtype=np.int32)
    thr = np.zeros((len(cascs), width))
    ns = np.zeros(len(cascs), dtype=np.int32)
    for c, (s, t) in enumerate(cascs):
        ns[c] = len(s)
        sm[c, : len(s)] = [index[m] for m in s]
        thr[c, : len(t)] = t
    return sm, thr, ns


def grid_configs_py(grids):
    """Grid-product enumeration (order documented in gridsweep.py)."""
    M = len(grids)
    rows_sm, rows_thr, rows_ns = [], [], []
    for k in range(1, M + 1):
        for combo in itertools.combinations(range(M), k):
            for ks in itertools.product(*[range(len(grids[m])) for m in combo[:-1]]):
                sm = list(combo) + [-1] * (M - k)
                thr = [float(grids[m][i]) for m, i in zip(combo[:-1], ks)] + [0.0] * (M - k + 1)
                rows_sm.append(sm)
                rows_thr.append(thr[:M])
                rows_ns.append(k)
    return (np.array(rows_sm, dtype=np.int32), np.array(rows_thr, dtype=np.float64),
            np.array(rows_ns, dtype=np.int32))


def certainty_tuples(seed: int = 11, n: int = 600, width: int = 6):
    rng = np.random.default_rng(seed)
    rows = rng.normal(size=(n, width))
    lens = rng.integers(1, width + 1, size=n).astype(np.int32)
    # duplicate maxima, exact ties, negatives, zeros
    dup = rng.random(n) < 0.2
    rows[dup, 1] = rows[dup, 0]
    rows[rng.random(n) < 0.05, :] = 0.0
    rows = np.round(rows, rng.integers(1, 8))
    return rows, lens


def logits_f32(seed: int, n: int, n_cls: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((n, n_cls)).astype(np.float32)
    boost = rng.integers(0, n_cls, size=n)
    x[np.arange(n), boost] += rng.uniform(0, 6, size=n).astype(np.float32)
    return x


def pareto_cases():
    rng = np.random.default_rng(5)
    cases = []
    for t in range(6):
        n = int(rng.integers(1, 300))
        acc = np.round(rng.random(n), int(rng.integers(1, 3)))
        cost = np.round(rng.uniform(0, 100, n), int(rng.integers(0, 2)))
        cases.append((acc, cost))
    return cases


def engine_cases():
    """Random plans (2-4 models, 1-3 replicas per model, 1-3 gears) and a
    batch of items at random stages for EngineState.finish_batch."""
    rng = np.random.default_rng(21)
    cases = []
    for t in range(8):
        n_models = int(rng.integers(2, 5))
        mids = [f"m{j}" for j in range(n_models)]
        n_rec = int(rng.integers(5, 60))
        cert = np.round(rng.random((n_rec, n_models)), 2)
        corr = (rng.random((n_rec, n_models)) < 0.6).astype(np.uint8)
        replicas = []
        for j, m in enumerate(mids):
            for r in range(int(rng.integers(1, 4))):
                replicas.append((f"{m}@d{r}", m, f"d{r}"))
        gears = []
        for g in range(int(rng.integers(1, 4))):
            k = int(rng.integers(1, n_models + 1))
            stages = sorted(rng.choice(n_models, size=k, replace=False).tolist())
            stages = [mids[i] for i in stages]
            thr = [float(np.round(rng.random(), 2)) for _ in stages[:-1]]
            weights = {}
            for m in stages:
                reps = [rid for rid, mm, _ in replicas if mm == m]
                w = np.round(rng.random(len(reps)) * 3, 1)
                if t == 3 and m == stages[-1]:
                    w[:] = 0.0  # all-zero weights: uniform integer draw
                weights[m] = {rid: float(x) for rid, x in zip(reps, w)}
            gears.append(dict(stages=stages, thresholds=thr, weights=weights))
        items = []
        for i in range(int(rng.integers(1, 40))):
            g = int(rng.integers(0, len(gears)))
            st = int(rng.integers(0, len(gears[g]["stages"])))
            items.append(dict(request_id=1000 * t + i, row=int(rng.integers(0, n_rec)),
                              stage=st, gear=g, arrival_us=int(rng.integers(0, 5000))))
        cases.append(dict(mids=mids, n_rec=n_rec, cert=cert, corr=corr, replicas=replicas,
                          gears=gears, items=items, now=10_000, seed=int(rng.integers(0, 99))))
    return cases


# ------------------------------------------------------------- replay ----
def bursty_counts(seconds: int, seed: int, base: float = 100.0, sigma: float = 0.7):
    """Per-second request counts of a bursty (Azure-like) series: lognormal
    levels, default_rng(seed)."""
    rng = np.random.default_rng(seed)
    return np.rint(base * rng.lognormal(0.0, sigma, seconds)).astype(np.int64) + 1


def trace_from_counts(counts):
    """A trace with counts[s] arrivals at the start of second s (input to
    scale_trace, which only reads the per-second counts)."""
    return np.repeat(np.arange(len(counts), dtype=np.int64) * 1_000_000, counts)


def replay_cases():
    """Engine replay scenarios (plain data; tests build reference or mirror
    objects from them).  Each exercises a different part of engine.run:
    gear switching under bursts, zero-weight stages (rng.integers draws),
    min queue lengths, multi-device dispatch order, probes without ticks,
    a t=0 burst (burst-throughput probe), a C7-like step trace."""
    def plan(models, replicas, gears, qps_max):
        return {"models": models, "replicas": replicas, "gears": gears, "qps_max": qps_max}

    m3 = {"n_models": 3, "cost_ratios": [1.0, 4.0, 16.0]}
    m4 = {"n_models": 4, "cost_ratios": [1.0, 4.0, 16.0, 64.0]}
    reps_a = [["m0@d0", "m0", "d0"], ["m1@d0", "m1", "d0"], ["m2@d1", "m2", "d1"],
              ["m0@d1", "m0", "d1"]]
    gears_a = [
        {"stages": ["m0", "m1", "m2"], "thresholds": [0.5, 0.6], "min_q": {"m0@d0": 2},
         "weights": {"m0": {"m0@d0": 3.0, "m0@d1": 1.0}, "m1": {"m1@d0": 1.0},
                     "m2": {"m2@d1": 1.0}}},
        {"stages": ["m0", "m2"], "thresholds": [0.7], "min_q": {},
         "weights": {"m0": {"m0@d0": 0.0, "m0@d1": 0.0}, "m2": {"m2@d1": 2.0}}},
    ]
    reps_c = [["m0@d0", "m0", "d0"], ["m1@d0", "m1", "d0"], ["m0@d1", "m0", "d1"],
              ["m2@d1", "m2", "d1"], ["m3@d2", "m3", "d2"], ["m1@d2", "m1", "d2"],
              ["m2@d2", "m2", "d2"]]
    gears_c = [
        {"stages": ["m0", "m1", "m2", "m3"], "thresholds": [0.55, 0.62, 0.7],
         "min_q": {"m3@d2": 2},
         "weights": {"m0": {"m0@d0": 1.0, "m0@d1": 1.0}, "m1": {"m1@d0": 2.0, "m1@d2": 1.0},
                     "m2": {"m2@d1": 1.0, "m2@d2": 0.5}, "m3": {"m3@d2": 1.0}}},
        {"stages": ["m0", "m2", "m3"], "thresholds": [0.6, 0.75], "min_q": {"m0@d0": 3},
         "weights": {"m0": {"m0@d0": 1.0, "m0@d1": 2.0}, "m2": {"m2@d1": 0.0, "m2@d2": 0.0},
                     "m3": {"m3@d2": 1.0}}},
        {"stages": ["m0", "m1"], "thresholds": [0.65], "min_q": {},
         "weights": {"m0": {"m0@d0": 1.0, "m0@d1": 1.0}, "m1": {"m1@d0": 1.0, "m1@d2": 3.0}}},
        {"stages": ["m0"], "thresholds": [], "min_q": {"m0@d0": 4, "m0@d1": 4},
         "weights": {"m0": {"m0@d0": 1.0, "m0@d1": 1.0}}},
    ]
    return {
        "bursty_two_gears": {"profiles": m3, "plan": plan(m3, reps_a, gears_a, 400.0),
                             "val": [500, 0.8, 1], "trace": {"bursty": [12, 5, 300.0]},
                             "seed": 7, "period": 100_000, "alpha": 8.0, "ticks": True,
                             "initial_gear": 0},
        "probe_no_ticks": {"profiles": m3, "plan": plan(m3, reps_a, gears_a[:1], 200.0),
                           "val": [300, 0.7, 2], "trace": {"constant": [200.0, 5.0]},
                           "seed": 11, "period": 100_000, "alpha": 8.0, "ticks": False,
                           "initial_gear": 0},
        "four_gears_overload": {"profiles": m4, "plan": plan(m4, reps_c, gears_c, 1000.0),
                                "val": [800, 0.8, 3], "trace": {"bursty": [10, 9, 900.0]},
                                "seed": 3, "period": 50_000, "alpha": 4.0, "ticks": True,
                                "initial_gear": 1},
        "burst_at_zero": {"profiles": m3, "plan": plan(m3, reps_a, gears_a[1:], 1.0),
                          "val": [400, 0.8, 4], "trace": {"zeros": [2000, 30_000_000]},
                          "seed": 5, "period": 100_000, "alpha": 8.0, "ticks": False,
                          "initial_gear": 0},
        "step_trace": {"profiles": m4, "plan": plan(m4, reps_c, gears_c, 160.0),
                       "val": [400, 0.9, 0], "trace": {"step": [[30.0, 6.0], [150.0, 6.0],
                                                                [30.0, 8.0]]},
                       "seed": 3, "period": 100_000, "alpha": 8.0, "ticks": True,
                       "initial_gear": 0},
    }
