"""Bind the reference `gearserve` package's hot path to the B200 library.

This is the reference-side binding INTEGRATION.md §2 describes, applied
in-process to an unmodified `gearserve` import (no reference file edited):

  gearserve.kernels.evaluate_encoded      (src/kernels.py:93-108)
      -> kernels.evaluate_encoded (gs_eval_encoded, bit-exact walk)
  gearserve.cascades.matrices             (src/cascades.py:44-63)
      -> one batched device certainty launch (gs_certainty), host copies
         cached on the ValidationSet exactly where the reference caches them
         (also the name engine.py imports, src/engine.py:22)
  gearserve.cascades.certainty            (src/cascades.py:20-28)
      -> gs_certainty (also the name serving.py imports, src/serving.py:25)
  gearserve.cascades.pareto_filter        (src/cascades.py:116-129)
      -> gs_pareto_generic (also the name planner.py imports, :25-33)
  gearserve.engine.EngineState.finish_batch (src/engine.py:355-383)
      -> the gate on the device, one packed H2D / kernel / D2H per batch
         (gs_stage_gate_packed); completions, queue appends and the shared
         Generator's draws in the reference's order.
  gearserve.cascades.sample_cascades      (src/cascades.py:166-193)
      -> the device sampler (gs_sample_cascades, numpy's stream reproduced)
         (also the name planner.py imports), with planner=True
  gearserve.planner.sp1_search_cascades   (src/planner.py:365-390), with
      planner=True -> the same steps, with every candidate's burst-throughput
         probe (_burst_throughput :329-357, one engine.run each in the
         reference) replayed in ONE device launch (replay.run_many) and put in
         the planner's own probe cache before its loop reads them.
  gearserve.engine.run (src/engine.py:452-520), with engine_run=True
      -> the whole virtual-clock event loop on the device (replay.py,
         gs_engine_run), which the planner's probes call too
         (src/planner.py:306, :348); wall-clock pacing (it sleeps in real
         time) and the batch log (record_batches) stay the reference's loop.

Everything that is not on the hot path (planner SP2-SP4, the LP, the event
loop, the threaded server, formats, CLI) stays the reference's own code.
`install()` returns the counters of calls routed to the library, so a test
can prove the GPU path actually ran.
"""

from __future__ import annotations

import importlib
from collections import Counter

import numpy as np
import torch

from . import _lib
from . import cascades as b200_cascades
from . import kernels as b200_kernels
from .stage import GateBatcher
from . import replay

CALLS: Counter = Counter()
_INSTALLED: dict = {}


def _evaluate_encoded(certainty, correct, stage_model, thresholds, n_stages, cost1):
    CALLS["evaluate_encoded"] += 1
    return b200_kernels.evaluate_encoded(certainty, correct, stage_model, thresholds,
                                         n_stages, cost1)


def _certainty(scores) -> float:
    CALLS["certainty"] += 1
    return b200_cascades.certainty(scores)


def _matrices(validation, profiles):
    """Reference cascades.matrices: same cache key, same error, same arrays."""
    key = profiles.model_ids
    cached = validation._matrix_cache.get(key)
    if cached is not None:
        return cached
    missing = set(key) - validation.model_ids
    if missing:
        raise ValueError(f"validation set lacks records for models {sorted(missing)}")
    CALLS["matrices"] += 1
    cert, corr = b200_cascades._device_matrices(validation, profiles)
    host = (cert.cpu().numpy(), corr.cpu().numpy())
    validation._matrix_cache[key] = host
    return host


def _pareto_filter(evals):
    CALLS["pareto_filter"] += 1
    return b200_cascades.pareto_filter(evals)


class _PlanGate:
    """Device view of one CompiledPlan: certainty / correct matrices and the
    per-gear (stage -> model, threshold, n_stages) tables of _CompiledGear
    (src/engine.py:175-193), plus the packed gate."""

    def __init__(self, comp):
        self.batcher = GateBatcher(torch.from_numpy(np.ascontiguousarray(comp.cert)),
                                   torch.from_numpy(np.ascontiguousarray(comp.corr)),
                                   capacity=max(8, max(comp.max_batch)))
        n = len(comp.gears)
        L = max(len(g.stage_model_idx) for g in comp.gears)
        self.model = np.zeros((n, L), dtype=np.int32)
        self.thr = np.zeros((n, L), dtype=np.float64)
        self.n_stages = np.zeros(n, dtype=np.int64)
        for gi, g in enumerate(comp.gears):
            k = len(g.stage_model_idx)
            self.model[gi, :k] = g.stage_model_idx
            self.thr[gi, : k - 1] = [float(t) for t in g.stage_thresholds[:-1]]
            self.n_stages[gi] = k


def _plan_gate(comp) -> _PlanGate:
    pg = getattr(comp, "_b200_gate", None)
    if pg is None or pg.batcher.cert.device.index != torch.cuda.current_device():
        pg = _PlanGate(comp)
        comp._b200_gate = pg
    return pg


def _make_finish_batch(engine_mod):
    RequestRecord = engine_mod.RequestRecord
    choose_weighted = engine_mod.choose_weighted

    def finish_batch(self, device_idx, items, now):
        """EngineState.finish_batch with the gate on the device (reference
        src/engine.py:355-383; same records, queue order and RNG draws)."""
        comp = self.compiled
        self.device_busy[device_idx] = False
        self.in_flight -= len(items)
        touched = {device_idx}
        if not items:
            return touched
        CALLS["finish_batch"] += 1
        pg = _plan_gate(comp)
        n = len(items)
        gear = np.fromiter((it.gear_idx for it in items), dtype=np.int64, count=n)
        stage = np.fromiter((it.stage for it in items), dtype=np.int64, count=n)
        rows = np.fromiter((it.row for it in items), dtype=np.int64, count=n)
        stop, correct, _ = pg.batcher.gate(rows, pg.model[gear, stage], pg.thr[gear, stage],
                                           stage == pg.n_stages[gear] - 1)
        for i, it in enumerate(items):
            if stop[i]:
                ok = bool(correct[i])
                self.request_records.append(RequestRecord(
                    request_id=it.request_id, arrival_us=it.arrival_us, completion_us=now,
                    stages_executed=it.stage + 1, correct=ok, gear_index=it.gear_idx))
                self.completed += 1
                self._window_latencies.append(now - it.arrival_us)
                self._window_correct += 1 if ok else 0
            else:
                g = comp.gears[it.gear_idx]
                it.stage += 1
                pos = choose_weighted(g.stage_cum_weights[it.stage], self.rng)
                ridx = int(g.stage_replica_idx[it.stage][pos])
                self.queues[ridx].append(it)
                touched.add(comp.device_of[ridx])
        return touched

    return finish_batch


def _make_run(engine_mod, reference_run):
    def run(plan, trace, validation, profiles, clock_mode="virtual", seed=None, config=None):
        """engine.run with the virtual-clock loop on the device."""
        if clock_mode not in ("virtual", "wall"):
            raise ValueError(f"clock_mode must be 'virtual' or 'wall', got {clock_mode!r}")
        if len(trace) == 0:
            raise ValueError("trace is empty")
        cfg = config or engine_mod.EngineConfig()
        if clock_mode == "wall" or cfg.record_batches:
            CALLS["run_reference_loop"] += 1
            return reference_run(plan, trace, validation, profiles, clock_mode=clock_mode,
                                 seed=seed, config=config)
        if seed is not None:
            cfg = engine_mod.replace(cfg, seed=seed)
        engine_mod.CompiledPlan(plan, profiles, validation)  # the reference's validation
        if not 0 <= cfg.initial_gear_index < len(plan.gears):
            raise ValueError(f"initial gear {cfg.initial_gear_index} out of range")
        CALLS["run"] += 1
        dp = replay.DevicePlan(plan, profiles, validation)
        job = replay.Job(dp, trace.arrivals, trace.duration_us, replay.EngineConfig(
            seed=cfg.seed, measure_period_us=cfg.measure_period_us, alpha=cfg.alpha,
            initial_gear_index=cfg.initial_gear_index, enable_ticks=cfg.enable_ticks))
        return replay.run_many([job])[0].to_sim_metrics(engine_mod)

    return run


def _make_sample_cascades(types_mod):
    def sample_cascades(profiles, grid, n_samples, rng_seed):
        """sample_cascades on the device, returned as reference Cascades."""
        if n_samples < 1:
            raise ValueError(f"n_samples must be >= 1, got {n_samples}")
        CALLS["sample_cascades"] += 1
        out = b200_cascades.sample_cascades_device(profiles, grid, n_samples, rng_seed)[0]
        ids = list(profiles.model_ids)
        sm, th, ns = (t.cpu().numpy() for t in (out.stage_model, out.thresholds, out.n_stages))
        return [types_mod.Cascade(stages=tuple(ids[int(m)] for m in sm[i, :ns[i]]),
                                  thresholds=tuple(float(x) for x in th[i, : ns[i] - 1]))
                for i in range(out.count)]

    return sample_cascades


def _burst_probes(planner_mod, types_mod, state, cascades) -> None:
    """Every uncached _burst_throughput probe (src/planner.py:329-357) of
    `cascades` replayed in one launch; results go into state._burst_cache
    under the planner's own key, computed as the reference computes them."""
    P = planner_mod
    placement = state.placement
    keys, jobs = [], []
    for c in cascades:
        key = (placement.signature(), c)
        if key in state._burst_cache or key in keys:
            continue
        if any(not placement.replicas_of(m) for m in c.stages):
            continue  # the reference's own path caches 0.0
        weights = {m: {r.replica_id: 1.0 for r in placement.replicas_of(m)} for m in c.stages}
        gear = P._build_gear(state, 0, placement=placement, cascade=c, weights=weights, q=1)
        plan = types_mod.GearPlan(placement=placement, slo=state.slo, qps_max=1.0, gears=(gear,))
        n = state.config.burst_probe_samples
        serial_us = sum(state.profiles[m].runtime_table[1] for m in c.stages)
        duration = n * serial_us * 2 + 1_000_000
        dp = replay.DevicePlan(plan, state.profiles, state.validation)
        keys.append(key)
        jobs.append(replay.Job(dp, np.zeros(n, dtype=np.int64), duration,
                               replay.EngineConfig(seed=state.seed, enable_ticks=False)))
    if not jobs:
        return
    CALLS["burst_probe_launches"] += 1
    CALLS["burst_probes"] += len(jobs)
    for key, res in zip(keys, replay.run_many(jobs)):
        if res.completed == 0:
            val = 0.0
        else:
            makespan = int(res.records["completion_us"].max())
            val = res.completed / (makespan / 1_000_000) if makespan > 0 else 0.0
        state._burst_cache[key] = val


def _make_sp1(planner_mod, types_mod):
    P = planner_mod

    def sp1_search_cascades(err, state):
        """SP1 (src/planner.py:365-390): sample, evaluate, Pareto, fallback
        singletons, then the candidates' burst probes -- all on the device,
        the probes in one batched replay launch."""
        state.counters["sp1"] += 1
        if not err.is_ok:
            raise P.UserInfeasible(
                "impossible to meet the SLO given the provided hardware resource: "
                + (err.reason or "all cascade downgrades exhausted"))
        sampled = P.sample_cascades(state.profiles, state.grid, state.config.n_samples,
                                    rng_seed=state.seed + state.counters["sp1"] - 1)
        evals = P.evaluate_cascades(sampled, state.validation, state.profiles)
        by_cascade = dict(zip(sampled, evals))
        keep = [c for c, _ in P.pareto_filter(list(by_cascade.items()))]
        singles = [(c, by_cascade[c]) for c in map(P._singleton, state.profiles.model_ids)]
        cheapest = min(singles, key=lambda p: (p[1].mean_cost, p[0].stages))[0]
        most_accurate = max(singles, key=lambda p: (p[1].accuracy, -p[1].mean_cost))[0]
        for c in [cheapest, most_accurate] + keep:
            if c not in state.candidate_cascades:
                state.candidate_cascades[c] = P.CandidateInfo(
                    cascade=c, eval=by_cascade[c], throughput_qps=0.0,
                    added_at_call=state.call_index)
        _burst_probes(P, types_mod, state, [i.cascade for i in state.candidate_cascades.values()])
        for info in state.candidate_cascades.values():
            info.throughput_qps = P._burst_throughput(state, info.cascade, state.placement)
        return P.PlannerError.ok(), state

    return sp1_search_cascades


def install(package: str = "gearserve", engine_gate: bool = True,
            engine_run: bool = False, planner: bool = False) -> Counter:
    """Route the reference package's hot path to the B200 library (no CPU
    fallback: the first routed call raises if the library or the GPU is
    missing).  Idempotent; returns the call counters."""
    if package in _INSTALLED:
        return CALLS
    _lib.load()
    kernels = importlib.import_module(f"{package}.kernels")
    cascades = importlib.import_module(f"{package}.cascades")
    engine = importlib.import_module(f"{package}.engine")
    planner = importlib.import_module(f"{package}.planner")
    serving = importlib.import_module(f"{package}.serving")
    saved = [(kernels, "evaluate_encoded", kernels.evaluate_encoded),
             (cascades, "certainty", cascades.certainty),
             (cascades, "matrices", cascades.matrices),
             (cascades, "pareto_filter", cascades.pareto_filter),
             (engine, "matrices", engine.matrices),
             (planner, "pareto_filter", planner.pareto_filter),
             (serving, "certainty", serving.certainty)]
    kernels.evaluate_encoded = _evaluate_encoded
    cascades.certainty = _certainty
    cascades.matrices = _matrices
    cascades.pareto_filter = _pareto_filter
    engine.matrices = _matrices
    planner.pareto_filter = _pareto_filter
    serving.certainty = _certainty
    if engine_gate:
        saved.append((engine.EngineState, "finish_batch", engine.EngineState.finish_batch))
        engine.EngineState.finish_batch = _make_finish_batch(engine)
    if engine_run:
        saved.append((engine, "run", engine.run))
        engine.run = _make_run(engine, engine.run)
    if planner:
        types_mod = importlib.import_module(f"{package}.types")
        saved += [(cascades, "sample_cascades", cascades.sample_cascades),
                  (planner, "sample_cascades", planner.sample_cascades),
                  (planner, "sp1_search_cascades", planner.sp1_search_cascades)]
        sampler = _make_sample_cascades(types_mod)
        cascades.sample_cascades = sampler
        planner.sample_cascades = sampler
        sp1 = _make_sp1(planner, types_mod)
        planner.sp1_search_cascades = sp1
        # the coordinate-descent loop holds the function in its table (:757-762)
        table = planner._SUBMODULES
        saved.append((table, 0, table[0]))
        table[0] = ("sp1", sp1)
    _INSTALLED[package] = saved
    return CALLS


def uninstall(package: str = "gearserve") -> None:
    for obj, name, value in reversed(_INSTALLED.pop(package, [])):
        if isinstance(obj, list):
            obj[name] = value
        else:
            setattr(obj, name, value)
