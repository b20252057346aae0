"""Trace replay on the device: engine.run in virtual-clock mode, many runs
per launch (csrc/gs_engine.cu, gs_engine_run).

Reference: gearserve.engine.run (/root/reference/pkg/src/gearserve/
engine.py:452-520) over EngineState (:267-449) and CompiledPlan (:196-235).
`run()` takes the reference's own arguments (plan, trace, validation,
profiles, seed, config) and returns the same metrics; `run_many()` replays
many (plan, trace, seed) jobs in ONE launch, one warp each -- the shape of
config 5 (a bursty trace replayed by independent replica groups) and of the
planner's simulator probes (_probe_range / _burst_throughput,
src/planner.py:293-356), which the reference runs one engine.run at a time.

Equality with the reference is by construction (same event order, numpy's
PCG64 stream on the device, the same f64 gate) and checked against goldens
captured from the reference (tests/test_gpu_replay.py).  Not supported:
wall-clock pacing (clock_mode="wall" sleeps in real time; nothing to
accelerate) and EngineConfig.record_batches (the batch log) -> ValueError.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .cascades import _device_matrices

US_PER_S = 1_000_000


class gs_engine_plan(ctypes.Structure):
    _fields_ = [("cert", ctypes.c_void_p), ("corr", ctypes.c_void_p), ("n_records", ctypes.c_int64),
                ("n_cols", ctypes.c_int32), ("n_replicas", ctypes.c_int32),
                ("n_devices", ctypes.c_int32), ("n_gears", ctypes.c_int32),
                ("max_stages", ctypes.c_int32), ("batch_cap", ctypes.c_int32),
                ("replica_device", ctypes.c_void_p), ("replica_model", ctypes.c_void_p),
                ("replica_rank", ctypes.c_void_p), ("model_max_batch", ctypes.c_void_p),
                ("model_runtime_us", ctypes.c_void_p), ("gear_n_stages", ctypes.c_void_p),
                ("gear_model", ctypes.c_void_p), ("gear_thr", ctypes.c_void_p),
                ("gear_rep_off", ctypes.c_void_p), ("gear_rep", ctypes.c_void_p),
                ("gear_cum", ctypes.c_void_p), ("gear_min_qlen", ctypes.c_void_p),
                ("qps_max", ctypes.c_double)]


class gs_engine_job(ctypes.Structure):
    _fields_ = [("plan", ctypes.c_void_p), ("arrivals", ctypes.c_void_p),
                ("n_arrivals", ctypes.c_int64), ("horizon_us", ctypes.c_int64),
                ("rng_state_hi", ctypes.c_uint64), ("rng_state_lo", ctypes.c_uint64),
                ("rng_inc_hi", ctypes.c_uint64), ("rng_inc_lo", ctypes.c_uint64),
                ("rng_has_uint32", ctypes.c_uint32), ("rng_uinteger", ctypes.c_uint32),
                ("initial_gear", ctypes.c_int32), ("enable_ticks", ctypes.c_int32),
                ("measure_period_us", ctypes.c_int64), ("alpha", ctypes.c_double),
                ("rings", ctypes.c_void_p), ("ring_cap", ctypes.c_int64),
                ("scratch", ctypes.c_void_p), ("records", ctypes.c_void_p),
                ("windows", ctypes.c_void_p), ("windows_cap", ctypes.c_int64),
                ("model_batches", ctypes.c_void_p), ("replica_counts", ctypes.c_void_p),
                ("result", ctypes.c_void_p)]


RECORD_DTYPE = np.dtype([("completion_us", np.int64), ("request_id", np.int32),
                         ("stages_executed", np.uint8), ("correct", np.uint8),
                         ("gear_index", np.uint16)])
WINDOW_DTYPE = np.dtype([("end_us", np.int64), ("measured_qps", np.float64),
                         ("first_stage_queue_len", np.int32), ("gear_before", np.int32),
                         ("candidate_gear", np.int32), ("gear_after", np.int32),
                         ("completed", np.int64), ("p95_us", np.int64), ("accuracy", np.float64)])
assert RECORD_DTYPE.itemsize == 16 and WINDOW_DTYPE.itemsize == 56
MAX_REPLICAS = 256
MAX_DEVICES = 64


@dataclass
class EngineConfig:
    """reference EngineConfig (src/engine.py:37-44)"""
    seed: int = 0
    measure_period_us: int = 100_000
    alpha: float = 8.0
    initial_gear_index: int = 0
    enable_ticks: bool = True
    record_batches: bool = False


class DevicePlan:
    """CompiledPlan (src/engine.py:196-235) as device tables: replicas in
    placement order, devices in first-appearance order, per gear the stage
    models, thresholds, replica lists (CSR) with np.cumsum'd load weights and
    per-replica minimum queue lengths; runtimes [model][batch]."""

    def __init__(self, plan, profiles, validation):
        dev = _lib.device()
        model_ids = list(profiles.model_ids)
        model_index = {m: i for i, m in enumerate(model_ids)}
        missing = {m for g in plan.gears for m in g.cascade.stages} - set(validation.model_ids)
        if missing:
            raise ValueError(f"validation set lacks models {sorted(missing)}")
        self.plan = plan
        self.model_ids = model_ids
        self.replicas = list(plan.placement.replicas)
        R = len(self.replicas)
        self.replica_index = {r.replica_id: i for i, r in enumerate(self.replicas)}
        self.devices: list[str] = []
        dindex: dict = {}
        for r in self.replicas:
            if r.device_id not in dindex:
                dindex[r.device_id] = len(self.devices)
                self.devices.append(r.device_id)
        if R > MAX_REPLICAS or len(self.devices) > MAX_DEVICES:
            raise ValueError(f"replay supports <= {MAX_REPLICAS} replicas on <= {MAX_DEVICES} "
                             "devices per plan")
        self.device_of = np.array([dindex[r.device_id] for r in self.replicas], dtype=np.int32)
        model_of = np.array([model_index[r.model_id] for r in self.replicas], dtype=np.int32)
        order = sorted(range(R), key=lambda i: self.replicas[i].replica_id)
        rank = np.empty(R, dtype=np.int32)
        rank[order] = np.arange(R, dtype=np.int32)
        self.max_batch = [profiles[m].max_profiled_batch for m in model_ids]
        cap = max(self.max_batch)
        self.batch_cap = cap
        runtime = np.zeros((len(model_ids), cap + 1), dtype=np.int64)
        for j, m in enumerate(model_ids):
            for b in range(1, self.max_batch[j] + 1):
                runtime[j, b] = profiles[m].runtime_us(b)
        G = len(plan.gears)
        L = max(g.cascade.n_stages for g in plan.gears)
        n_st = np.zeros(G, dtype=np.int32)
        gmodel = np.zeros((G, L), dtype=np.int32)
        gthr = np.zeros((G, L), dtype=np.float64)
        off = np.zeros((G, L + 1), dtype=np.int32)
        reps, cums = [], []
        minq = np.ones((G, R), dtype=np.int32)
        for gi, gear in enumerate(plan.gears):
            casc = gear.cascade
            n_st[gi] = casc.n_stages
            for s, m in enumerate(casc.stages):
                off[gi, s] = len(reps)
                gmodel[gi, s] = model_index[m]
                if s < casc.n_stages - 1:
                    gthr[gi, s] = float(casc.thresholds[s])
                idxs = [i for i, r in enumerate(self.replicas) if r.model_id == m]
                if not idxs:
                    raise ValueError(f"gear {gi}: no replica of {m!r}")
                w = np.array([gear.load_weights[m].get(self.replicas[i].replica_id, 0.0)
                              for i in idxs])
                reps.extend(idxs)
                cums.extend(np.cumsum(w).tolist())
            off[gi, casc.n_stages:] = len(reps)
            for rid, q in gear.min_queue_length.items():
                minq[gi, self.replica_index[rid]] = int(q)
        cert, corr = _device_matrices(validation, profiles)
        self.cert, self.corr = cert.contiguous(), corr.contiguous()
        self.n_records = int(self.cert.shape[0])
        t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a)).to(dev, dt)  # noqa: E731
        self._keep = [t(self.device_of, torch.int32), t(model_of, torch.int32),
                      t(rank, torch.int32), t(np.array(self.max_batch), torch.int32),
                      t(runtime, torch.int64), t(n_st, torch.int32), t(gmodel, torch.int32),
                      t(gthr, torch.float64), t(off, torch.int32),
                      t(np.array(reps, dtype=np.int32), torch.int32),
                      t(np.array(cums, dtype=np.float64), torch.float64), t(minq, torch.int32)]
        k = self._keep
        st = gs_engine_plan(
            self.cert.data_ptr(), self.corr.data_ptr(), self.n_records, int(self.cert.shape[1]),
            R, len(self.devices), G, L, cap, k[0].data_ptr(), k[1].data_ptr(), k[2].data_ptr(),
            k[3].data_ptr(), k[4].data_ptr(), k[5].data_ptr(), k[6].data_ptr(), k[7].data_ptr(),
            k[8].data_ptr(), k[9].data_ptr(), k[10].data_ptr(), k[11].data_ptr(),
            float(plan.qps_max))
        raw = np.frombuffer(bytes(st), dtype=np.uint8)
        self.struct = torch.from_numpy(raw.copy()).to(dev)
        self.n_gears = G


def _rng_words(seed) -> tuple[int, int, int, int, int, int]:
    """numpy default_rng(seed)'s PCG64 state as (state hi, lo, inc hi, lo,
    has_uint32, uinteger)."""
    st = np.random.default_rng(seed).bit_generator.state
    s, inc = int(st["state"]["state"]), int(st["state"]["inc"])
    m = (1 << 64) - 1
    return s >> 64, s & m, inc >> 64, inc & m, int(st["has_uint32"]), int(st["uinteger"])


@dataclass
class ReplayResult:
    """Device replay outputs in columnar form (numpy)."""
    arrivals: int
    completed: int
    in_flight: int
    records: np.ndarray            # RECORD_DTYPE [completed], completion order
    arrival_us: np.ndarray         # [n_arrivals] the trace
    windows: np.ndarray            # WINDOW_DTYPE [n_windows]
    model_batches: np.ndarray      # [n_models, batch_cap + 1]
    routed: np.ndarray             # [R] submits routed to each replica
    queue_len: np.ndarray          # [R] queue lengths at the horizon
    rng_state: tuple               # (state, has_uint32, uinteger) after the run
    plan: DevicePlan = field(repr=False)
    period_us: int = 100_000

    def latencies_us(self) -> np.ndarray:
        r = self.records
        return r["completion_us"] - self.arrival_us[r["request_id"]]

    def to_sim_metrics(self, engine_mod=None):
        """The reference's SimMetrics (src/engine.py:76-108; _collect_metrics
        :422-449), built with the reference's own record classes when
        engine_mod (gearserve.engine) is given, else with this module's."""
        mod = engine_mod
        RequestRecord = mod.RequestRecord if mod else _RequestRecord
        WindowRecord = mod.WindowRecord if mod else _WindowRecord
        SimMetrics = mod.SimMetrics if mod else _SimMetrics
        r = self.records
        per_request = [RequestRecord(request_id=int(i), arrival_us=int(self.arrival_us[i]),
                                     completion_us=int(c), stages_executed=int(s),
                                     correct=bool(k), gear_index=int(g))
                       for i, c, s, k, g in zip(r["request_id"], r["completion_us"],
                                                r["stages_executed"], r["correct"],
                                                r["gear_index"])]
        windows = []
        for w in self.windows:
            windows.append(WindowRecord(
                end_us=int(w["end_us"]), measured_qps=float(w["measured_qps"]),
                first_stage_queue_len=int(w["first_stage_queue_len"]),
                gear_before=int(w["gear_before"]), candidate_gear=int(w["candidate_gear"]),
                gear_after=int(w["gear_after"]), observed_range=int(w["candidate_gear"]),
                completed=int(w["completed"]),
                p95_us=None if w["p95_us"] < 0 else int(w["p95_us"]),
                accuracy=None if math.isnan(w["accuracy"]) else float(w["accuracy"])))
        range_windows: dict = {}
        range_completed: dict = {}
        for w in windows:
            range_windows[w.observed_range] = range_windows.get(w.observed_range, 0) + 1
            range_completed[w.observed_range] = range_completed.get(w.observed_range, 0) + \
                w.completed
        period_s = self.period_us / US_PER_S
        throughput = {k: range_completed[k] / (n * period_s) for k, n in range_windows.items()}
        total_w = sum(range_windows.values())
        fractions = {k: n / total_w for k, n in range_windows.items()} if total_w else {}
        per_model = {}
        for j, m in enumerate(self.plan.model_ids):
            hist = {int(b): int(c) for b, c in enumerate(self.model_batches[j]) if c}
            if hist:
                per_model[m] = hist
        return SimMetrics(
            arrivals=self.arrivals, completed=self.completed,
            backlogged=self.arrivals - self.completed,
            latencies_us=self.latencies_us().astype(np.int64), per_request=per_request,
            per_model_batches=per_model, per_range_throughput=throughput,
            per_range_time_fraction=fractions, windows=windows,
            queue_len_at_horizon={rep.replica_id: int(q) for rep, q in
                                  zip(self.plan.replicas, self.queue_len)},
            in_flight_at_horizon=self.in_flight, batch_log=None)


@dataclass(frozen=True)
class _RequestRecord:
    request_id: int
    arrival_us: int
    completion_us: int
    stages_executed: int
    correct: bool
    gear_index: int


@dataclass(frozen=True)
class _WindowRecord:
    end_us: int
    measured_qps: float
    first_stage_queue_len: int
    gear_before: int
    candidate_gear: int
    gear_after: int
    observed_range: int
    completed: int
    p95_us: int | None
    accuracy: float | None


@dataclass
class _SimMetrics:
    arrivals: int
    completed: int
    backlogged: int
    latencies_us: np.ndarray
    per_request: list
    per_model_batches: dict
    per_range_throughput: dict
    per_range_time_fraction: dict
    windows: list
    queue_len_at_horizon: dict
    in_flight_at_horizon: int
    batch_log: list | None = None


@dataclass
class Job:
    """One replay: a compiled plan, a trace, a seed and the engine config."""
    plan: DevicePlan
    arrivals: np.ndarray | torch.Tensor
    horizon_us: int
    config: EngineConfig = field(default_factory=EngineConfig)


class _JobBuffers:
    def __init__(self, job: Job, dev):
        cfg = job.config
        if cfg.record_batches:
            raise ValueError("the device replay does not keep the batch log (record_batches)")
        if not 0 <= cfg.initial_gear_index < job.plan.n_gears:
            raise ValueError(f"initial gear {cfg.initial_gear_index} out of range")
        arr = job.arrivals
        self.arr = arr.to(dev, torch.int64).contiguous() if isinstance(arr, torch.Tensor) else \
            torch.from_numpy(np.ascontiguousarray(arr, dtype=np.int64)).to(dev)
        n = int(self.arr.numel())
        if n >= (1 << 31) - 1:
            raise ValueError("replay supports < 2^31 arrivals per job")
        self.n = n
        p = job.plan
        R = len(p.replicas)
        self.n_windows_cap = (job.horizon_us // cfg.measure_period_us
                              if cfg.enable_ticks and cfg.measure_period_us > 0 else 0)
        i32 = dict(dtype=torch.int32, device=dev)
        i64 = dict(dtype=torch.int64, device=dev)
        m = max(n, 1)
        # a ring per replica queue, each able to hold every request
        self.rings = torch.empty(R * m, **i64)
        self.scratch = torch.empty(m, **i64)
        self.records = torch.empty(m * 2, **i64)           # 16-byte records
        self.windows = torch.empty(max(self.n_windows_cap, 1) * 7, **i64)  # 56-byte windows
        self.batches = torch.empty(len(p.model_ids) * (p.batch_cap + 1), **i64)
        self.counts = torch.empty(2 * R, **i64)
        self.result = torch.empty(8, **i64)
        w = _rng_words(cfg.seed)
        self.struct = gs_engine_job(
            p.struct.data_ptr(), self.arr.data_ptr() if n else None, n, int(job.horizon_us),
            w[0], w[1], w[2], w[3], w[4], w[5], int(cfg.initial_gear_index),
            1 if cfg.enable_ticks else 0, int(cfg.measure_period_us), float(cfg.alpha),
            self.rings.data_ptr(), m, self.scratch.data_ptr(),
            self.records.data_ptr(), self.windows.data_ptr(), int(self.n_windows_cap),
            self.batches.data_ptr(), self.counts.data_ptr(), self.result.data_ptr())


class Prepared:
    """Device buffers and the descriptor table of a batch of jobs: the host
    work (allocation, trace and plan uploads) done once, so run() is one
    kernel launch and can be repeated (every launch rewrites the outputs)."""

    def __init__(self, jobs: list[Job]):
        dev = _lib.device()
        self.jobs = list(jobs)
        self.bufs = [_JobBuffers(j, dev) for j in self.jobs]
        raw = b"".join(bytes(b.struct) for b in self.bufs)
        self.table = torch.from_numpy(np.frombuffer(raw, dtype=np.uint8).copy()).to(dev) \
            if raw else None

    def run(self) -> "Prepared":
        """One gs_engine_run launch over every job, on the current stream."""
        if self.bufs:
            _lib.check(_lib.load().gs_engine_run(self.table.data_ptr(), len(self.bufs),
                                                 _lib.stream_ptr()), "engine replay")
        return self

    def results(self) -> list["ReplayResult"]:
        return [collect(j, b) for j, b in zip(self.jobs, self.bufs)]


def launch(jobs: list[Job]) -> list[_JobBuffers]:
    """Enqueue every job's replay in ONE gs_engine_run launch on the current
    stream; returns the per-job device buffers (read them with collect())."""
    prep = Prepared(jobs).run()
    for b in prep.bufs:
        b.table = prep.table  # keep the descriptor table alive with the buffers
    return prep.bufs


def collect(job: Job, b: _JobBuffers) -> ReplayResult:
    res = b.result.cpu().numpy()
    arrivals, completed, in_flight, n_win = (int(x) for x in res[:4])
    if n_win > b.n_windows_cap:
        raise RuntimeError("window capacity exceeded")
    rec = b.records.cpu().numpy().view(RECORD_DTYPE)[:completed].copy()
    win = b.windows.cpu().numpy().view(np.uint8)[: n_win * 56].view(WINDOW_DTYPE).copy()
    p = job.plan
    counts = b.counts.cpu().numpy().reshape(-1, 2)
    state = (int(np.uint64(res[4])) << 64) | int(np.uint64(res[5]))
    return ReplayResult(
        arrivals=arrivals, completed=completed, in_flight=in_flight, records=rec,
        arrival_us=b.arr.cpu().numpy(), windows=win,
        model_batches=b.batches.cpu().numpy().reshape(len(p.model_ids), p.batch_cap + 1),
        routed=counts[:, 0].copy(), queue_len=counts[:, 1].copy(),
        rng_state=(state, int(res[6]), int(res[7])), plan=p,
        period_us=int(job.config.measure_period_us))


def run_many(jobs: list[Job]) -> list[ReplayResult]:
    """Replay every job in one launch and collect the results."""
    bufs = launch(jobs)
    return [collect(j, b) for j, b in zip(jobs, bufs)]


def run(plan, trace, validation, profiles, clock_mode: str = "virtual", seed: int | None = None,
        config: EngineConfig | None = None, engine_mod=None):
    """engine.run (src/engine.py:452-520), virtual clock, on the device.
    Returns the reference-shaped SimMetrics (engine_mod: build it with the
    reference's own classes)."""
    if clock_mode != "virtual":
        raise ValueError("the device replay runs the virtual clock only")
    if len(trace) == 0:
        raise ValueError("trace is empty")
    cfg = config or EngineConfig()
    if seed is not None:
        cfg = EngineConfig(seed=seed, measure_period_us=cfg.measure_period_us, alpha=cfg.alpha,
                           initial_gear_index=cfg.initial_gear_index,
                           enable_ticks=cfg.enable_ticks, record_batches=cfg.record_batches)
    dp = DevicePlan(plan, profiles, validation)
    job = Job(dp, trace.arrivals, trace.duration_us, cfg)
    return run_many([job])[0].to_sim_metrics(engine_mod)


# ---------------------------------------------------------------- traces --
def scale_trace(trace, target_max_qps: float):
    """formats.scale_trace (src/formats.py:137-150): per-second counts scaled
    so the busiest second carries target_max_qps (np.rint), each second's
    arrivals spread evenly inside it; the horizon keeps the trace's seconds."""
    from .types import WorkloadTrace
    if target_max_qps <= 0:
        raise ValueError(f"target max QPS must be positive, got {target_max_qps}")
    arr = np.asarray(trace.arrivals, dtype=np.int64)
    counts = np.bincount(arr // US_PER_S, minlength=trace.duration_us // US_PER_S) \
        if arr.size else np.zeros(0, dtype=np.int64)
    if counts.size == 0 or counts.max() == 0:
        raise ValueError("cannot scale an empty trace")
    new = np.rint(counts * (target_max_qps / counts.max())).astype(np.int64)
    sec = np.repeat(np.arange(new.size, dtype=np.int64), new)
    first = np.repeat(np.cumsum(new) - new, new)
    k = np.arange(sec.size, dtype=np.int64) - first          # position inside its second
    per = np.repeat(new, new)
    arrivals = sec * US_PER_S + (k * US_PER_S) // np.maximum(per, 1)
    return WorkloadTrace(arrivals, duration_us=int(counts.size) * US_PER_S)


def split_round_robin(trace, groups: int):
    """Split a trace over `groups` independent replica groups (request i goes
    to group i % groups): each group is one engine state, one replay job."""
    from .types import WorkloadTrace
    return [WorkloadTrace(trace.arrivals[g::groups], duration_us=trace.duration_us)
            for g in range(groups)]
