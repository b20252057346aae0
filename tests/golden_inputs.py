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
