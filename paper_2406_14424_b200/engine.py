"""Batched cascade stage step for the serving engine.

Mirrors the routing slice of gearserve.engine
(/root/reference/pkg/src/gearserve/engine.py):
  _CompiledGear (:175-193)  -> GearTables: per-gear stage model, threshold,
                               replica list and cumulative load weights
  choose_weighted (:238-245) -> route(): the same numpy Generator draws, made
                               once per forwarded item in batch order
  _Item (:256-264)           -> Item
  EngineState.finish_batch (:355-383) -> StageRouter.finish_batch

The gate itself (last stage, or cert[row, m] >= thr) and the order-preserving
compaction of the forwarded items run on the device (stage.stage_gate over the
compiled certainty / correct matrices, the analogue of CompiledPlan.cert /
corr, :217).  Replica choice stays on the host: it must consume the engine's
numpy Generator exactly as the reference does, one rng.random() per
forwarded item (or one rng.integers when a stage's weights are all zero), and
rng.random(n) yields the same stream as n scalar draws, so whole runs of
forwarded items are drawn at once.
"""

from __future__ import annotations

from bisect import bisect_right
from collections import deque
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .stage import GateBatcher


@dataclass
class Item:
    """One in-flight request (reference _Item)."""

    request_id: int
    row: int
    stage: int
    gear_idx: int
    arrival_us: int


@dataclass(frozen=True)
class Completion:
    """RequestRecord fields the stage step produces (reference :368-376)."""

    request_id: int
    arrival_us: int
    completion_us: int
    stages_executed: int
    correct: bool
    gear_index: int


class GearTables:
    """Dense per-gear routing tables.

    stage_models[g]   model column of each stage of gear g
    thresholds[g]     forwarding threshold per stage (last stage: None)
    replicas[g][s]    replica indices serving stage s (placement order)
    cum_weights[g][s] np.cumsum of their load weights
    """

    def __init__(self, stage_models, thresholds, replicas, cum_weights):
        self.stage_models = [list(map(int, s)) for s in stage_models]
        self.thresholds = [list(t) for t in thresholds]
        self.replicas = [[np.asarray(r, dtype=np.int64) for r in g] for g in replicas]
        self.cum_weights = [[np.asarray(c, dtype=np.float64) for c in g] for g in cum_weights]
        n = len(self.stage_models)
        if not (len(self.thresholds) == len(self.replicas) == len(self.cum_weights) == n):
            raise ValueError("gear tables disagree on the number of gears")
        L = max(len(s) for s in self.stage_models)
        self.max_stages = L
        # flattened [gear, stage] lookups for the device gate
        self._model = np.full((n, L), -1, dtype=np.int32)
        self._thr = np.zeros((n, L), dtype=np.float64)
        self._n_stages = np.zeros(n, dtype=np.int64)
        for g, (sm, th) in enumerate(zip(self.stage_models, self.thresholds)):
            if len(th) != len(sm) or th[-1] is not None:
                raise ValueError("thresholds need one entry per stage, None at the last")
            self._model[g, : len(sm)] = sm
            self._thr[g, : len(sm) - 1] = th[:-1]
            self._n_stages[g] = len(sm)

    @classmethod
    def from_gears(cls, gears, replica_models, model_index):
        """Build from reference-shaped gears: objects with .cascade.stages,
        .cascade.thresholds and .load_weights[model][replica_id]; replica_models
        is the placement order [(replica_id, model_id)]."""
        sm, th, rep, cum = [], [], [], []
        for g in gears:
            stages = g.cascade.stages
            sm.append([model_index[m] for m in stages])
            th.append(list(g.cascade.thresholds) + [None])
            rs, cs = [], []
            for m in stages:
                idx = [i for i, (_, mm) in enumerate(replica_models) if mm == m]
                w = np.array([g.load_weights[m].get(replica_models[i][0], 0.0) for i in idx])
                rs.append(np.array(idx, dtype=np.int64))
                cs.append(np.cumsum(w))
            rep.append(rs)
            cum.append(cs)
        return cls(sm, th, rep, cum)


def choose_weighted(cum_weights: np.ndarray, rng: np.random.Generator) -> int:
    """One weighted draw (reference engine.choose_weighted)."""
    total = cum_weights[-1]
    if total <= 0.0:
        return int(rng.integers(len(cum_weights)))
    x = rng.random() * total
    return int(np.searchsorted(cum_weights, x, side="right").clip(0, len(cum_weights) - 1))


def route(tables: GearTables, gears: np.ndarray, stages: np.ndarray,
          rng: np.random.Generator) -> np.ndarray:
    """Replica index for each forwarded item (in batch order), drawing from
    rng exactly as a sequence of choose_weighted calls would."""
    n = len(gears)
    out = np.empty(n, dtype=np.int64)
    totals = np.array([tables.cum_weights[g][s][-1] for g, s in zip(gears, stages)])
    i = 0
    while i < n:
        if totals[i] <= 0.0:  # uniform integer draw, one at a time
            g, s = int(gears[i]), int(stages[i])
            pos = int(rng.integers(len(tables.cum_weights[g][s])))
            out[i] = tables.replicas[g][s][pos]
            i += 1
            continue
        j = i
        while j < n and totals[j] > 0.0:
            j += 1
        x = rng.random(j - i) * totals[i:j]  # same doubles as j-i scalar draws
        keys = gears[i:j] * tables.max_stages + stages[i:j]
        for key in np.unique(keys):
            sel = np.flatnonzero(keys == key)
            g, s = divmod(int(key), tables.max_stages)
            cum = tables.cum_weights[g][s]
            pos = np.searchsorted(cum, x[sel], side="right").clip(0, len(cum) - 1)
            out[i + sel] = tables.replicas[g][s][pos]
        i = j
    return out


class StageRouter:
    """Queues, completions and the batched finish_batch transition.

    Holds the state finish_batch touches in the reference EngineState
    (queues per replica, request records, counters, the shared Generator);
    the device certainty/correct matrices are uploaded once.
    """

    def __init__(self, tables: GearTables, cert, corr, replica_device, seed: int = 0,
                 rng: np.random.Generator | None = None, near_keep: int = 4096):
        self.tables = tables
        self.cert = _lib.to_device(cert, torch.float64)
        self.corr = _lib.to_device(corr, torch.uint8)
        self.gate = GateBatcher(self.cert, self.corr)
        self.replica_device = np.asarray(replica_device, dtype=np.int64)
        self.queues = [deque() for _ in range(len(self.replica_device))]
        self.rng = rng if rng is not None else np.random.default_rng(seed)
        self.completed: list[Completion] = []
        self.n_completed = 0
        self.in_flight = 0
        self.window_latencies: list[int] = []
        self.window_correct = 0
        # request ids gated within 1e-6 of their threshold: the most recent
        # near_keep of them (bounded for long-running routers), and a count
        self.near_threshold: deque[int] = deque(maxlen=near_keep)
        self.n_near_threshold = 0
        # Python-list copies of the tables for small batches (numpy's per-call
        # overhead exceeds the work at the reference's 4-8 items)
        G = len(tables.stage_models)
        self._model_l = [[int(tables._model[g, s]) for s in range(tables.max_stages)] for g in range(G)]
        self._thr_l = [[float(tables._thr[g, s]) for s in range(tables.max_stages)] for g in range(G)]
        self._nst_l = [int(tables._n_stages[g]) for g in range(G)]
        self._cum_l = [[[float(x) for x in c] for c in tables.cum_weights[g]] for g in range(G)]
        self._rep_l = [[[int(x) for x in r] for r in tables.replicas[g]] for g in range(G)]
        self._dev_l = [int(d) for d in self.replica_device]

    SMALL = 256  # batches up to this size take the list path

    def _finish_small(self, device_idx: int, items: list[Item], now: int) -> set[int]:
        """finish_batch for a small batch: the same gate call and the same
        draws (one rng.random() per forwarded item in batch order, or
        rng.integers for a zero-weight stage: route's stream), over lists."""
        touched = {device_idx}
        ml, tl, nst = self._model_l, self._thr_l, self._nst_l
        rows, model, thr, last = [], [], [], []
        for it in items:
            g, st = it.gear_idx, it.stage
            rows.append(it.row)
            model.append(ml[g][st])
            thr.append(tl[g][st])
            last.append(st == nst[g] - 1)
        stop, correct, near = self.gate.gate_small(rows, model, thr, last)
        if near:
            self.n_near_threshold += len(near)
            self.near_threshold.extend(items[i].request_id for i in near)
        rng, cl, rl, dl = self.rng, self._cum_l, self._rep_l, self._dev_l
        for i, it in enumerate(items):
            if stop[i]:
                ok = bool(correct[i])
                self.completed.append(Completion(it.request_id, it.arrival_us, now, it.stage + 1, ok,
                                                 it.gear_idx))
                self.n_completed += 1
                self.window_latencies.append(now - it.arrival_us)
                self.window_correct += 1 if ok else 0
        for i, it in enumerate(items):  # forwards in batch order
            if stop[i]:
                continue
            g, st = it.gear_idx, it.stage + 1
            cum = cl[g][st]
            if cum[-1] <= 0.0:
                pos = int(rng.integers(len(cum)))
            else:
                pos = min(bisect_right(cum, rng.random() * cum[-1]), len(cum) - 1)
            r = rl[g][st][pos]
            it.stage = st
            self.queues[r].append(it)
            touched.add(dl[r])
        return touched

    def finish_batch(self, device_idx: int, items: list[Item], now: int) -> set[int]:
        """Complete certain items, forward the rest (batch order kept);
        returns the devices to re-scan.  Same outcome as the reference."""
        self.in_flight -= len(items)
        touched = {device_idx}
        if not items:
            return touched
        if len(items) <= self.SMALL:
            return self._finish_small(device_idx, items, now)
        t = self.tables
        gear = np.fromiter((it.gear_idx for it in items), dtype=np.int64, count=len(items))
        stage = np.fromiter((it.stage for it in items), dtype=np.int64, count=len(items))
        rows = np.fromiter((it.row for it in items), dtype=np.int64, count=len(items))
        model = t._model[gear, stage]
        thr = t._thr[gear, stage]
        last = stage == t._n_stages[gear] - 1
        # one H2D of the packed items, the device gate, one D2H of the outcome
        stop, correct, near = self.gate.gate(rows, model, thr, last)
        fwd = np.flatnonzero(~stop)  # batch order, as the kernel compacts them
        self.n_near_threshold += len(near)
        self.near_threshold.extend(items[i].request_id for i in near)
        for i in np.flatnonzero(stop):
            it = items[i]
            ok = bool(correct[i])
            self.completed.append(Completion(it.request_id, it.arrival_us, now, it.stage + 1, ok,
                                             it.gear_idx))
            self.n_completed += 1
            self.window_latencies.append(now - it.arrival_us)
            self.window_correct += 1 if ok else 0
        if len(fwd):
            nxt = stage[fwd] + 1
            replicas = route(t, gear[fwd], nxt, self.rng)
            for i, r in zip(fwd, replicas):
                it = items[i]
                it.stage += 1
                self.queues[int(r)].append(it)
                touched.add(int(self.replica_device[r]))
        return touched
