"""CPU oracle — TEST INFRASTRUCTURE ONLY.

Restatements of the reference (gearserve, /root/reference/pkg/src/gearserve)
for the hot path, used as the checker by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference arm.  Nothing in the product
package imports this module.

Pinned: tests/test_oracle.py checks every function here against golden
vectors captured from the reference itself (tests/golden/make_golden.py,
run where /root/reference is importable) — see DESIGN.md "Oracle".

Functions and the reference lines they restate:
  evaluate_encoded      kernels._evaluate_numba        kernels.py:39-62   (C, oracle_eval.c)
  grid_configs          enumeration of the grid product (documented in gridsweep.py)
  certainty             cascades.certainty              cascades.py:20-28
  margin_rows           cascades.certainty over a matrix (f64 after promotion)
  max_softmax_rows / entropy_rows   extension definitions (no reference; unpinned)
  pareto_keep           cascades.pareto_filter          cascades.py:116-129
  choose_weighted       engine.choose_weighted          engine.py:238-245
  finish_batch          EngineState.finish_batch        engine.py:355-383
  stage_step            gate + stable compaction of finish_batch on score rows
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
BUILD = HERE / "_build"
LIB = BUILD / "liboracle.so"


def build(force: bool = False) -> Path:
    """gcc the C restatement (OpenMP, no FP contraction)."""
    src = HERE / "oracle_eval.c"
    if not force and LIB.exists() and LIB.stat().st_mtime >= src.stat().st_mtime:
        return LIB
    BUILD.mkdir(exist_ok=True)
    tmp = LIB.with_suffix(".so.tmp")
    subprocess.run(["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fPIC", "-shared",
                    str(src), "-o", str(tmp)], check=True)
    os.replace(tmp, LIB)
    return LIB


_lib = None


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(str(LIB))
        P = ctypes.c_void_p
        lib.oracle_evaluate_encoded.argtypes = [P, P, ctypes.c_int64, ctypes.c_int32, P, P, P,
                                                ctypes.c_int64, ctypes.c_int32, P, P, P, P,
                                                ctypes.c_int32]
        lib.oracle_evaluate_encoded.restype = None
        lib.oracle_grid_n_configs.argtypes = [ctypes.c_int32, P]
        lib.oracle_grid_n_configs.restype = ctypes.c_int64
        lib.oracle_grid_configs.argtypes = [ctypes.c_int32, P, P, ctypes.c_int64,
                                            ctypes.c_int64, P, P, P]
        lib.oracle_grid_configs.restype = ctypes.c_int
        lib.oracle_max_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def max_threads() -> int:
    return int(_load().oracle_max_threads())


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


# ------------------------------------------------------------ the walk ----
def evaluate_encoded(certainty, correct, stage_model, thresholds, n_stages, cost1,
                     n_threads: int = 1):
    """(accuracy, mean_cost, forward_frac) exactly as _evaluate_numba."""
    cert = np.ascontiguousarray(certainty, dtype=np.float64)
    corr = np.ascontiguousarray(correct, dtype=np.uint8)
    sm = np.ascontiguousarray(stage_model, dtype=np.int32)
    thr = np.ascontiguousarray(thresholds, dtype=np.float64)
    ns = np.ascontiguousarray(n_stages, dtype=np.int32)
    c1 = np.ascontiguousarray(cost1, dtype=np.float64)
    n_casc, L = sm.shape
    acc = np.zeros(n_casc)
    cost = np.zeros(n_casc)
    frac = np.zeros((n_casc, L))
    if n_casc:
        _load().oracle_evaluate_encoded(_p(cert), _p(corr), cert.shape[0], cert.shape[1],
                                        _p(sm), _p(thr), _p(ns), n_casc, L, _p(c1), _p(acc),
                                        _p(cost), _p(frac), int(n_threads))
    return acc, cost, frac


def walk_python(certainty, correct, stage_model, thresholds, n_stages, cost1):
    """Pure-Python restatement (small cases only) — pins the C port."""
    n_rec = certainty.shape[0]
    n_casc, L = stage_model.shape
    acc = np.zeros(n_casc)
    cost = np.zeros(n_casc)
    frac = np.zeros((n_casc, L))
    for c in range(n_casc):
        ns = int(n_stages[c])
        n_correct = 0
        for r in range(n_rec):
            for s in range(ns):
                m = int(stage_model[c, s])
                frac[c, s] += 1.0
                if s == ns - 1 or certainty[r, m] >= thresholds[c, s]:
                    n_correct += int(correct[r, m])
                    break
        for s in range(ns):
            f = frac[c, s] / n_rec
            frac[c, s] = f
            cost[c] += f * cost1[int(stage_model[c, s])]
        acc[c] = n_correct / n_rec
    return acc, cost, frac


def grid_n_configs(grid_len) -> int:
    gl = np.ascontiguousarray(grid_len, dtype=np.int32)
    return int(_load().oracle_grid_n_configs(len(gl), _p(gl)))


def grid_configs(grids, begin: int = 0, count: int | None = None):
    """Encoded cascades (stage_model, thresholds, n_stages) of the grid
    product configs [begin, begin+count)."""
    gl = np.ascontiguousarray([len(g) for g in grids], dtype=np.int32)
    flat = np.ascontiguousarray(np.concatenate([np.asarray(g, np.float64) for g in grids]))
    total = grid_n_configs(gl)
    if count is None:
        count = total - begin
    M = len(grids)
    sm = np.empty((count, M), dtype=np.int32)
    thr = np.empty((count, M), dtype=np.float64)
    ns = np.empty(count, dtype=np.int32)
    if count:
        _load().oracle_grid_configs(M, _p(gl), _p(flat), begin, count, _p(sm), _p(thr), _p(ns))
    return sm, thr, ns


# ------------------------------------------------------------ certainty ---
def certainty(scores) -> float:
    """cascades.certainty: top minus second of the sorted scores; a single
    score is returned as is; empty raises ValueError."""
    if len(scores) == 0:
        raise ValueError("certainty of empty scores")
    if len(scores) == 1:
        return float(scores[0])
    top, second = sorted(scores, reverse=True)[:2]
    return float(top - second)


def margin_rows(scores: np.ndarray, row_len=None) -> np.ndarray:
    """Eq. 5 per row on the values promoted to f64 (vectorised)."""
    x = np.asarray(scores).astype(np.float64)
    n, c = x.shape
    if row_len is not None:
        row_len = np.asarray(row_len)
        x = x.copy()
        x[np.arange(c)[None, :] >= row_len[:, None]] = -np.inf
    else:
        row_len = np.full(n, c)
    if c == 1:
        return x[:, 0].copy()
    part = -np.partition(-x, 1, axis=1)[:, :2]
    out = part[:, 0] - part[:, 1]
    single = row_len == 1
    out[single] = x[single, 0]
    return out


def max_softmax_rows(scores: np.ndarray) -> np.ndarray:
    """Extension: max softmax probability = 1 / sum exp(x - max), f64."""
    x = np.asarray(scores).astype(np.float64)
    m = x.max(axis=1, keepdims=True)
    return 1.0 / np.exp(x - m).sum(axis=1)


def entropy_rows(scores: np.ndarray) -> np.ndarray:
    """Extension: 1 - H(softmax(x)) / ln(n_cls), f64 (1.0 for n_cls == 1)."""
    x = np.asarray(scores).astype(np.float64)
    n_cls = x.shape[1]
    if n_cls == 1:
        return np.ones(x.shape[0])
    d = x - x.max(axis=1, keepdims=True)
    e = np.exp(d)
    s = e.sum(axis=1)
    t = (e * d).sum(axis=1)
    H = np.log(s) - t / s
    return 1.0 - H / np.log(n_cls)


CERT_ORACLES = {"margin": margin_rows, "max_softmax": max_softmax_rows,
                "entropy": entropy_rows}


# ---------------------------------------------------------------- pareto --
def pareto_keep(acc, cost) -> np.ndarray:
    """Boolean keep mask with pareto_filter's exact semantics (O(n log n)):
    keep e iff acc_e is the max of its cost group and exceeds the best
    accuracy over strictly cheaper groups."""
    acc = np.asarray(acc, dtype=np.float64)
    cost = np.asarray(cost, dtype=np.float64)
    n = acc.size
    if n == 0:
        return np.zeros(0, dtype=bool)
    order = np.lexsort((-acc, cost))
    keep = np.zeros(n, dtype=bool)
    best_cheaper = -np.inf
    i = 0
    while i < n:
        j = i
        c = cost[order[i]]
        while j < n and cost[order[j]] == c:
            j += 1
        group = order[i:j]
        gmax = acc[group].max()
        if gmax > best_cheaper:
            keep[group[acc[group] == gmax]] = True
        best_cheaper = max(best_cheaper, gmax)
        i = j
    return keep


def pareto_keep_quadratic(acc, cost) -> np.ndarray:
    """Literal O(n^2) restatement of pareto_filter (small n)."""
    n = len(acc)
    keep = np.ones(n, dtype=bool)
    for i in range(n):
        for j in range(n):
            if (acc[j] >= acc[i] and cost[j] <= cost[i]
                    and (acc[j] > acc[i] or cost[j] < cost[i])):
                keep[i] = False
                break
    return keep


# ------------------------------------------------------------ stage step --
def choose_weighted(cum_weights: np.ndarray, rng: np.random.Generator) -> int:
    """engine.choose_weighted: one rng.random() scaled by the total, or
    rng.integers(len) when every weight is zero."""
    total = cum_weights[-1]
    if total <= 0.0:
        return int(rng.integers(len(cum_weights)))
    x = rng.random() * total
    return int(np.searchsorted(cum_weights, x, side="right").clip(0, len(cum_weights) - 1))


def stage_step(cert: np.ndarray, thr: np.ndarray, is_last=None, near_eps: float = 1e-6,
               payload: np.ndarray | None = None):
    """finish_batch's gate on a batch: stop mask, deferred rows in batch
    order, rows within near_eps of their threshold (non-last), gathered
    payload."""
    cert = np.asarray(cert, dtype=np.float64)
    thr = np.broadcast_to(np.asarray(thr, dtype=np.float64), cert.shape)
    last = np.zeros(cert.shape, dtype=bool) if is_last is None else np.asarray(is_last, bool)
    stop = last | (cert >= thr)
    deferred = np.flatnonzero(~stop)
    near = np.flatnonzero(~last & (np.abs(cert - thr) <= near_eps))
    nxt = None if payload is None else payload[deferred]
    return stop, deferred, near, nxt


def finish_batch(items, gears, cert, corr, rng, now):
    """EngineState.finish_batch restated on plain data.

    items: list of dicts {request_id, row, stage, gear, arrival_us}
    gears: list of dicts {stage_model: [..], thresholds: [.., None],
           replica_idx: [array per stage], cum_weights: [array per stage]}
    Returns (completed, forwarded): completed = [(request_id, correct,
    stages_executed, latency)], forwarded = [(item position, replica)] in
    batch order; rng is advanced exactly as the reference advances it.
    """
    completed, forwarded = [], []
    for pos, it in enumerate(items):
        g = gears[it["gear"]]
        m = g["stage_model"][it["stage"]]
        thr = g["thresholds"][it["stage"]]
        last = it["stage"] == len(g["stage_model"]) - 1
        if last or cert[it["row"], m] >= thr:
            completed.append((it["request_id"], bool(corr[it["row"], m]), it["stage"] + 1,
                              now - it["arrival_us"]))
        else:
            nxt = it["stage"] + 1
            p = choose_weighted(g["cum_weights"][nxt], rng)
            forwarded.append((pos, int(g["replica_idx"][nxt][p])))
    return completed, forwarded


def load_validation_jsonl(path):
    """Restatement of the reference reader (src/formats.py:75-97): json.loads
    per non-blank line, scores through float(), correct through bool(),
    sample_id through int().  Returns (sample_ids, {model: [scores tuples]},
    {model: [bool]}) in file order."""
    import json
    ids, scores, correct = [], {}, {}
    with open(path) as f:
        for lineno, line in enumerate(f, start=1):
            line = line.strip()
            if not line:
                continue
            try:
                doc = json.loads(line)
                outs = {mid: (tuple(float(s) for s in out["scores"]), bool(out["correct"]))
                        for mid, out in doc["models"].items()}
                sid = int(doc["sample_id"])
            except (json.JSONDecodeError, KeyError, TypeError, ValueError) as e:
                raise ValueError(f"{path}: line {lineno}: {e}")
            ids.append(sid)
            for mid, (sc, ok) in outs.items():
                scores.setdefault(mid, []).append(sc)
                correct.setdefault(mid, []).append(ok)
    return ids, scores, correct


def grid_values(cert_column, levels: int) -> tuple:
    """build_threshold_grid's per-model grid (src/cascades.py:157-162) with
    numpy on the host: {0} U np.quantile(col, k/levels), sorted."""
    qs = [k / levels for k in range(1, levels)]
    quants = np.quantile(np.asarray(cert_column, dtype=np.float64), qs)
    return tuple(sorted({0.0} | {float(q) for q in quants}))


# ------------------------------------------------------------- PCG64 ---
class Pcg64:
    """numpy's default_rng bit generator (PCG64, XSL-RR output of the
    advanced state) with its buffered 32-bit half, restated in Python: the
    stream gs_engine.cu / the device sampler reproduce.  Test infrastructure."""

    MULT = 0x2360ED051FC65DA44385DF649FCCF645
    M128 = (1 << 128) - 1

    def __init__(self, seed):
        st = np.random.default_rng(seed).bit_generator.state
        self.s, self.inc = int(st["state"]["state"]), int(st["state"]["inc"])
        self.has32, self.u32 = int(st["has_uint32"]), int(st["uinteger"])

    def state(self):
        return (self.s, self.has32, self.u32)

    def next64(self) -> int:
        self.s = (self.s * self.MULT + self.inc) & self.M128
        x = ((self.s >> 64) ^ self.s) & ((1 << 64) - 1)
        r = self.s >> 122
        return ((x >> r) | (x << ((64 - r) & 63))) & ((1 << 64) - 1)

    def next32(self) -> int:
        if self.has32:
            self.has32 = 0
            return self.u32
        n = self.next64()
        self.has32, self.u32 = 1, n >> 32
        return n & 0xFFFFFFFF

    def random(self) -> float:
        return (self.next64() >> 11) * (1.0 / 9007199254740992.0)

    def bounded(self, rng: int) -> int:
        """numpy's Lemire sampler on [0, rng] (rng < 2^32)."""
        if rng == 0:
            return 0
        excl = rng + 1
        m = self.next32() * excl
        if (m & 0xFFFFFFFF) < excl:
            thr = (0xFFFFFFFF - rng) % excl
            while (m & 0xFFFFFFFF) < thr:
                m = self.next32() * excl
        return m >> 32

    def integers(self, lo: int, hi: int | None = None) -> int:
        if hi is None:
            lo, hi = 0, lo
        return lo + self.bounded(hi - 1 - lo)


def sample_cascades_pcg(order_grid_len, n_samples: int, seed: int):
    """sample_cascades (src/cascades.py:166-193) restated on Pcg64: returns
    the list of (cost ranks, threshold grid indices) in output order --
    the algorithm gs_sampler.cu runs.  order_grid_len[r] is the grid length
    of the model at cost rank r.  Test infrastructure."""
    M = len(order_grid_len)
    g = Pcg64(seed)
    out = [((r,), ()) for r in range(M)]
    seen = set(out)
    for _ in range(n_samples):
        k = g.integers(1, M + 1)
        taken, pick = set(), []
        for j in range(M - k, M):
            v = g.bounded(j)
            if v not in taken:
                taken.add(v)
                pick.append(v)
            else:
                taken.add(j)
                pick.append(j)
        for i in range(k - 1, 0, -1):
            jj = g.bounded(i)
            pick[jj], pick[i] = pick[i], pick[jj]
        ranks = tuple(sorted(pick))
        gidx = tuple(g.bounded(order_grid_len[r] - 1) for r in ranks[:-1])
        if (ranks, gidx) not in seen:
            seen.add((ranks, gidx))
            out.append((ranks, gidx))
    return out, g.state()


# --------------------------------------------------------- engine.run ---
def engine_run(plan, trace, cert, corr, runtime, max_batch, model_index, seed: int = 0,
               period_us: int = 100_000, alpha: float = 8.0, initial_gear: int = 0,
               enable_ticks: bool = True):
    """engine.run (src/engine.py:452-520) in virtual-clock mode restated over
    plain arrays: the event heap, submit (:299-319), scan_device /
    choose_dispatch (:321-353, :248-253), finish_batch (:355-383), tick /
    maybe_switch_gear (:389-410, :123-133), nearest-rank p95 (:111-120).
    plan: objects with .placement.replicas (replica_id, model_id, device_id),
    .gears (cascade.stages / thresholds, min_queue_length, load_weights) and
    .qps_max; runtime[model][batch] µs; returns a dict of arrays.  Test
    infrastructure (the checker of gs_engine.cu and the config-5 CPU
    baseline); the reference is pure Python, so this loop is its cost model."""
    import heapq
    import math
    from collections import deque
    reps = list(plan.placement.replicas)
    R = len(reps)
    devices, dindex = [], {}
    for r in reps:
        if r.device_id not in dindex:
            dindex[r.device_id] = len(devices)
            devices.append(r.device_id)
    device_of = [dindex[r.device_id] for r in reps]
    model_of = [model_index[r.model_id] for r in reps]
    rid_of = [r.replica_id for r in reps]
    gears = []
    for g in plan.gears:
        st = g.cascade.stages
        ridx = [[i for i, r in enumerate(reps) if r.model_id == m] for m in st]
        cum = [np.cumsum([g.load_weights[m].get(reps[i].replica_id, 0.0) for i in idx])
               for m, idx in zip(st, ridx)]
        minq = [1] * R
        for rid, q in g.min_queue_length.items():
            minq[rid_of.index(rid)] = q
        gears.append(([model_index[m] for m in st], list(g.cascade.thresholds) + [None],
                      ridx, cum, minq))
    rng = np.random.default_rng(seed)

    def choose(cum):
        total = cum[-1]
        if total <= 0.0:
            return int(rng.integers(len(cum)))
        x = rng.random() * total
        return int(np.searchsorted(cum, x, side="right").clip(0, len(cum) - 1))

    queues = [deque() for _ in range(R)]
    busy = [False] * len(devices)
    item_stage, item_gear = {}, {}
    arrivals_t = np.asarray(trace.arrivals, dtype=np.int64)
    n_rec = cert.shape[0]
    cur = initial_gear
    rec, wins = [], []
    batches = {}
    st = {"arrivals": 0, "completed": 0, "in_flight": 0}
    win = {"arr": 0, "lat": [], "ok": 0}
    heap, seq = [], 0
    horizon = trace.duration_us
    if enable_ticks:
        t = period_us
        while t <= horizon:
            heapq.heappush(heap, (t, 1, seq, "tick", None))
            seq += 1
            t += period_us
    nxt = 0
    if len(arrivals_t):
        heapq.heappush(heap, (int(arrivals_t[0]), 2, seq, "arrival", 0))
        seq += 1
        nxt = 1
    while heap:
        t, _, _, kind, arg = heapq.heappop(heap)
        if t > horizon:
            break
        if kind == "arrival":
            rid = arg
            g = gears[cur]
            item_stage[rid], item_gear[rid] = 0, cur
            ridx = int(g[2][0][choose(g[3][0])])
            queues[ridx].append(rid)
            st["arrivals"] += 1
            win["arr"] += 1
            touched = {device_of[ridx]}
            if nxt < len(arrivals_t):
                heapq.heappush(heap, (int(arrivals_t[nxt]), 2, seq, "arrival", nxt))
                seq += 1
                nxt += 1
        elif kind == "complete":
            d, items = arg
            busy[d] = False
            st["in_flight"] -= len(items)
            touched = {d}
            for rid in items:
                g = gears[item_gear[rid]]
                s = item_stage[rid]
                m = g[0][s]
                last = s == len(g[0]) - 1
                row = rid % n_rec
                if last or cert[row, m] >= g[1][s]:
                    ok = bool(corr[row, m])
                    rec.append((rid, int(arrivals_t[rid]), t, s + 1, int(ok), item_gear[rid]))
                    st["completed"] += 1
                    win["lat"].append(t - int(arrivals_t[rid]))
                    win["ok"] += 1 if ok else 0
                else:
                    item_stage[rid] = s + 1
                    ridx = int(g[2][s + 1][choose(g[3][s + 1])])
                    queues[ridx].append(rid)
                    touched.add(device_of[ridx])
        else:
            qps = win["arr"] / (period_us / 1_000_000)
            q0 = sum(len(queues[r]) for r in gears[cur][2][0])
            cand = min(int(math.floor(qps * len(gears) / plan.qps_max)), len(gears) - 1)
            after = cur if (cand < cur and qps < alpha * q0) else cand
            lat = win["lat"]
            p95 = -1
            if lat:
                arr = np.sort(np.asarray(lat))
                p95 = int(arr[max(1, math.ceil(95 / 100 * arr.size)) - 1])
            wins.append((t, qps, q0, cur, cand, after, len(lat), p95,
                         (win["ok"] / len(lat)) if lat else float("nan")))
            cur = after
            win = {"arr": 0, "lat": [], "ok": 0}
            touched = set(range(len(devices)))
        for d in sorted(touched):
            if busy[d]:
                continue
            cands = [(item_stage[queues[r][0]], -len(queues[r]), rid_of[r], r) for r in range(R)
                     if device_of[r] == d and queues[r] and len(queues[r]) >= gears[cur][4][r]]
            if not cands:
                continue
            r = min(cands)[3]
            m = model_of[r]
            size = min(len(queues[r]), max_batch[m])
            items = [queues[r].popleft() for _ in range(size)]
            busy[d] = True
            st["in_flight"] += size
            batches[(m, size)] = batches.get((m, size), 0) + 1
            heapq.heappush(heap, (t + int(runtime[m][size]), 0, seq, "complete", (d, items)))
            seq += 1
    return {"records": np.array(rec, dtype=np.int64).reshape(-1, 6),
            "windows": wins, "arrivals": st["arrivals"], "completed": st["completed"],
            "in_flight": st["in_flight"], "queue_len": [len(q) for q in queues],
            "batches": batches, "rng_state": rng.bit_generator.state}
