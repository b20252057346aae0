"""Drop-in for gearserve.cascades (/root/reference/pkg/src/gearserve/cascades.py).

Same public names, arguments, return types and errors as the reference:
certainty (:20-28), CascadeEval (:31-41), matrices (:44-63),
encode_cascades (:66-79), evaluate_cascades / evaluate_cascade (:82-106),
model_qps_demand (:109-113), pareto_filter (:116-129), ThresholdGrid /
build_threshold_grid (:132-163), sample_cascades (:166-193).

What moved to the GPU: certainty of score rows (gs_certainty, margin =
Eq. 5 bit-exact), the matrices ingest (one batched certainty launch instead
of the reference's per-record Python loop; the device copies are cached next
to the host copies), the cascade walk (gs_eval_encoded), and the Pareto
filter (gs_pareto_generic).  Host-side numpy remains only for marshalling
(encode_cascades), the threshold-grid quantiles and the seeded cascade
sampler, whose outputs must follow numpy's own quantile / Generator streams
(SURVEY §8f rows 3-4).

New here: sweep_grid(), the full cascade x threshold-grid product scored on
the device (gridsweep.GridSweep), with an exact Pareto reduction.
"""

from __future__ import annotations

import ctypes

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib, kernels
from .gridsweep import GridSweep
from .types import Cascade, ProfileSet, ValidationArrays, ValidationSet


# ------------------------------------------------------------- certainty --
def certainty_rows(scores, row_len=None, kind: str = "margin") -> torch.Tensor:
    """Certainty of every row of a score matrix [n, n_cls] (f32/f64/bf16,
    numpy or torch) on the device; returns a CUDA f64 tensor [n].
    row_len (optional [n] int) gives ragged lengths for padded rows."""
    if kind not in _lib.CERT_KINDS:
        raise ValueError(f"unknown certainty kind {kind!r}")
    if isinstance(scores, np.ndarray):
        dt = {np.dtype(np.float32): torch.float32, np.dtype(np.float64): torch.float64}.get(
            scores.dtype, torch.float64)
        s = _lib.to_device(scores, dt)
    else:
        s = _lib.to_device(scores, scores.dtype if scores.dtype in _lib.DTYPES else torch.float64)
    if s.ndim != 2:
        raise ValueError("scores must be [n_rows, n_cls]")
    n, c = int(s.shape[0]), int(s.shape[1])
    out = torch.empty(n, dtype=torch.float64, device=s.device)
    if n == 0:
        return out
    if c == 0:
        raise ValueError("certainty of empty scores")
    rl = None
    if row_len is not None:
        rl = _lib.to_device(np.asarray(row_len, dtype=np.int32), torch.int32)
        if int(rl.min()) < 1:
            raise ValueError("certainty of empty scores")
        if int(rl.max()) > c:
            raise ValueError("row length exceeds the score matrix width")
    lib = _lib.load()
    rc = lib.gs_certainty(s.data_ptr(), _lib.DTYPES[s.dtype], n, c, _lib.row_stride(s),
                          _lib.ptr(rl), _lib.CERT_KINDS[kind], out.data_ptr(),
                          _lib.stream_ptr())
    _lib.check(rc, "certainty")
    return out


def certainty(scores) -> float:
    """Prediction certainty: highest score minus second-highest; a single
    score is returned as is.  Empty scores raise ValueError."""
    if len(scores) == 0:
        raise ValueError("certainty of empty scores")
    row = np.asarray([float(x) for x in scores], dtype=np.float64)[None, :]
    return float(certainty_rows(row).item())


@dataclass(frozen=True)
class CascadeEval:
    """Offline metrics of one cascade on one validation set; mean_cost is
    the forward-fraction-weighted sum of batch-1 runtimes (µs)."""

    accuracy: float
    mean_cost: float
    forward_fraction: dict[str, float]


# --------------------------------------------------------------- matrices --
def _device_matrices(validation, profiles: ProfileSet):
    """(cert, corr) as CUDA tensors [n, M] in profile order, cached."""
    key = ("device",) + tuple(profiles.model_ids)
    hit = validation._matrix_cache.get(key)
    if hit is not None:
        return hit
    order = profiles.model_ids
    missing = set(order) - set(validation.model_ids)
    if missing:
        raise ValueError(f"validation set lacks records for models {sorted(missing)}")
    if isinstance(validation, ValidationArrays):
        cols = [validation.model_ids_ordered.index(m) for m in order]
        corr = _lib.to_device(np.asarray(validation.correct)[:, cols] != 0, torch.uint8) \
            if not isinstance(validation.correct, torch.Tensor) else \
            _lib.to_device((validation.correct[:, cols] != 0).to(torch.uint8), torch.uint8)
        if validation.certainty is not None:
            c = validation.certainty
            c = c[:, cols] if isinstance(c, torch.Tensor) else np.asarray(c)[:, cols]
            cert = _lib.to_device(c, torch.float64)
        else:
            rl = validation.row_len or {}
            cert = torch.stack([certainty_rows(validation.scores[m], row_len=rl.get(m))
                                for m in order], dim=1)
            cert = cert.contiguous()
    else:
        n, m_count = len(validation), len(order)
        lens = np.empty((n, m_count), dtype=np.int32)
        corr_h = np.empty((n, m_count), dtype=np.uint8)
        for i, rec in enumerate(validation.records):
            for j, mid in enumerate(order):
                out = rec.outputs[mid]
                lens[i, j] = len(out.scores)
                corr_h[i, j] = 1 if out.correct else 0
        width = int(lens.max())
        pad = np.zeros((n * m_count, width), dtype=np.float64)
        flat = lens.reshape(-1)
        for i, rec in enumerate(validation.records):
            for j, mid in enumerate(order):
                sc = rec.outputs[mid].scores
                pad[i * m_count + j, : len(sc)] = sc
        cert = certainty_rows(pad, row_len=None if np.all(flat == width) else flat)
        cert = cert.view(n, m_count)
        corr = _lib.to_device(corr_h, torch.uint8)
    validation._matrix_cache[key] = (cert, corr)
    return cert, corr


def matrices(validation, profiles: ProfileSet) -> tuple[np.ndarray, np.ndarray]:
    """(certainty, correct) matrices [n_records, n_models] in profile order,
    cached on the validation set (reference cascades.py:44-63)."""
    key = profiles.model_ids
    cached = validation._matrix_cache.get(key)
    if cached is not None:
        return cached
    cert, corr = _device_matrices(validation, profiles)
    host = (cert.cpu().numpy(), corr.cpu().numpy())
    validation._matrix_cache[key] = host
    return host


# ----------------------------------------------------------- evaluation --
def encode_cascades(cascades: list[Cascade], profiles: ProfileSet):
    """Pack cascades into the padded arrays the kernel takes
    (stage_model -1 padded, thresholds 0 padded, n_stages)."""
    max_len = max(c.n_stages for c in cascades)
    n = len(cascades)
    stage_model = np.full((n, max_len), -1, dtype=np.int32)
    thresholds = np.zeros((n, max_len), dtype=np.float64)
    n_stages = np.zeros(n, dtype=np.int32)
    index = {m: profiles.index(m) for m in profiles.model_ids}
    for ci, c in enumerate(cascades):
        k = c.n_stages
        n_stages[ci] = k
        stage_model[ci, :k] = [index[m] for m in c.stages]
        if k > 1:
            thresholds[ci, : k - 1] = c.thresholds
    return stage_model, thresholds, n_stages


def evaluate_cascades(cascades: list[Cascade], validation,
                      profiles: ProfileSet) -> list[CascadeEval]:
    if not cascades:
        return []
    for c in cascades:
        for mid in c.stages:
            if mid not in profiles:
                raise ValueError(f"cascade stage {mid!r} has no profile")
    cert, corr = _device_matrices(validation, profiles)
    stage_model, thresholds, n_stages = encode_cascades(cascades, profiles)
    cost1 = profiles.cost1()
    acc, cost, frac = kernels.evaluate_encoded_device(
        cert, corr, _lib.to_device(stage_model, torch.int32),
        _lib.to_device(thresholds, torch.float64), _lib.to_device(n_stages, torch.int32),
        _lib.to_device(cost1, torch.float64))
    acc, cost, frac = acc.cpu().numpy(), cost.cpu().numpy(), frac.cpu().numpy()
    out = []
    for ci, c in enumerate(cascades):
        ff = {mid: float(frac[ci, si]) for si, mid in enumerate(c.stages)}
        out.append(CascadeEval(accuracy=float(acc[ci]), mean_cost=float(cost[ci]),
                               forward_fraction=ff))
    return out


def evaluate_cascade(cascade: Cascade, validation, profiles: ProfileSet) -> CascadeEval:
    return evaluate_cascades([cascade], validation, profiles)[0]


def model_qps_demand(ev: CascadeEval, total_qps: float) -> dict[str, float]:
    """Per-model demand: forward fraction times total cascade QPS."""
    if total_qps < 0:
        raise ValueError(f"total_qps must be >= 0, got {total_qps}")
    return {m: f * total_qps for m, f in ev.forward_fraction.items()}


def pareto_filter(evals: list[tuple[Cascade, CascadeEval]]) -> list[tuple[Cascade, CascadeEval]]:
    """Keep entries no other entry dominates (accuracy >=, cost <=, one
    strict); exact ties survive; input order is kept."""
    if not evals:
        return []
    acc = np.array([ev.accuracy for _, ev in evals], dtype=np.float64)
    cost = np.array([ev.mean_cost for _, ev in evals], dtype=np.float64)
    keep = pareto_mask(acc, cost).cpu().numpy()
    return [e for e, k in zip(evals, keep) if k]


def pareto_mask(accuracy, mean_cost) -> torch.Tensor:
    """Device Pareto mask (u8 [n]) of float (accuracy, cost) points."""
    a = _lib.to_device(accuracy, torch.float64)
    c = _lib.to_device(mean_cost, torch.float64)
    n = int(a.numel())
    keep = torch.empty(n, dtype=torch.uint8, device=a.device)
    if n:
        rc = _lib.load().gs_pareto_generic(a.data_ptr(), c.data_ptr(), n, keep.data_ptr(),
                                           _lib.stream_ptr())
        _lib.check(rc, "pareto_filter")
    return keep


# ---------------------------------------------------------- grids, sampler --
@dataclass(frozen=True)
class ThresholdGrid:
    """Candidate thresholds per model, strictly increasing, starting at 0."""

    per_model: dict[str, tuple[float, ...]]

    def __post_init__(self) -> None:
        for mid, vals in self.per_model.items():
            if len(vals) == 0:
                raise ValueError(f"{mid}: empty threshold grid")
            if vals[0] != 0.0:
                raise ValueError(f"{mid}: grid must start at 0, got {vals[0]}")
            for a, b in zip(vals, vals[1:]):
                if not b > a:
                    raise ValueError(f"{mid}: grid not strictly increasing at {b}")


def quantiles(column, qs) -> np.ndarray:
    """np.quantile(column, qs) (numpy "linear", bit-exact) computed on the
    device (gs_quantiles: a radix select of the needed order statistics +
    numpy's interpolation arithmetic).
    column: a 1-D numpy array or CUDA tensor (any stride)."""
    qs = np.ascontiguousarray(np.asarray(qs, dtype=np.float64).reshape(-1))
    col = column if isinstance(column, torch.Tensor) else torch.from_numpy(
        np.ascontiguousarray(np.asarray(column, dtype=np.float64)))
    col = _lib.to_device(col, torch.float64) if col.device.type != "cuda" or \
        col.dtype != torch.float64 else col
    if col.ndim != 1 or col.numel() == 0:
        raise ValueError("quantiles of an empty or non-1-D column")
    n = int(col.numel())
    lib = _lib.load()
    nbytes = ctypes.c_size_t()
    _lib.check(lib.gs_quantiles_workspace(n, qs.size, ctypes.byref(nbytes)), "quantiles")
    ws = _lib.workspace(nbytes.value)
    out = torch.empty(max(qs.size, 1), dtype=torch.float64, device=col.device)
    rc = lib.gs_quantiles(col.data_ptr(), n, int(col.stride(0)), qs.ctypes.data, qs.size,
                          out.data_ptr(), ws.data_ptr(), ws.numel(), _lib.stream_ptr())
    _lib.check(rc, "quantiles")
    return out[: qs.size].cpu().numpy()


def grid_values(cert_column, levels: int) -> tuple[float, ...]:
    """{0} U quantiles k/levels (numpy linear), sorted (reference :157-162);
    the quantiles are taken on the device."""
    qs = [k / levels for k in range(1, levels)]
    quants = quantiles(cert_column, qs)
    return tuple(sorted({0.0} | {float(q) for q in quants}))


def build_threshold_grid(validation, profiles: ProfileSet, levels: int = 10) -> ThresholdGrid:
    """Per-model grids: 0 plus the certainty quantiles k/levels, k=1..levels-1."""
    if levels < 2:
        raise ValueError(f"levels must be >= 2, got {levels}")
    cert, _ = _device_matrices(validation, profiles)
    return ThresholdGrid(per_model={mid: grid_values(cert[:, j], levels)
                                    for j, mid in enumerate(profiles.model_ids)})


def sample_cascades(profiles: ProfileSet, grid: ThresholdGrid, n_samples: int,
                    rng_seed: int) -> list[Cascade]:
    """All singletons (cheap to expensive) then n_samples random model
    subsets ordered by (batch-1 runtime, index) with thresholds drawn from
    the grid; duplicates dropped in order.  Same numpy Generator stream as
    the reference (:166-193), so the same seed gives the same list."""
    if n_samples < 1:
        raise ValueError(f"n_samples must be >= 1, got {n_samples}")
    order = sorted(profiles.model_ids,
                   key=lambda m: (profiles[m].runtime_table[1], profiles.index(m)))
    rng = np.random.default_rng(rng_seed)
    out = [Cascade(stages=(m,), thresholds=()) for m in order]
    seen = set(out)
    n_models = len(order)
    for _ in range(n_samples):
        k = int(rng.integers(1, n_models + 1))
        pick = rng.choice(n_models, size=k, replace=False)
        stages = tuple(order[i] for i in sorted(pick))
        thrs = tuple(float(rng.choice(grid.per_model[m])) for m in stages[:-1])
        c = Cascade(stages=stages, thresholds=thrs)
        if c not in seen:
            seen.add(c)
            out.append(c)
    return out


# -------------------------------------------------------------- full grid --
@dataclass
class GridFront:
    """Pareto front of a full-grid sweep: cascades with their evals, in
    enumeration order, plus the sweep size."""

    cascades: list[Cascade]
    evals: list[CascadeEval]
    config_index: np.ndarray
    n_configs: int


def sweep_grid(validation, profiles: ProfileSet, grid: ThresholdGrid) -> GridFront:
    """Score the whole cascade x threshold-grid product on the device and
    return its exact Pareto front.  Models are walked cheap to expensive
    (batch-1 runtime, then profile index), as sample_cascades orders them."""
    order = sorted(profiles.model_ids,
                   key=lambda m: (profiles[m].runtime_table[1], profiles.index(m)))
    cols = [profiles.index(m) for m in order]
    cert, corr = _device_matrices(validation, profiles)
    cert, corr = cert[:, cols].contiguous(), corr[:, cols].contiguous()
    cost1 = profiles.cost1()[cols]
    sweep = GridSweep(cert, corr, [np.asarray(grid.per_model[m]) for m in order], cost1)
    idx, res = sweep.pareto()
    idx_h = idx.cpu().numpy()
    local = idx - res.config_begin
    acc = res.accuracy[local].cpu().numpy()
    cost = res.mean_cost[local].cpu().numpy()
    frac = res.forward_frac[local].cpu().numpy()
    cascs = sweep.cascades(idx, order)
    evals = [CascadeEval(accuracy=float(acc[i]), mean_cost=float(cost[i]),
                         forward_fraction={m: float(frac[i, s]) for s, m in enumerate(c.stages)})
             for i, c in enumerate(cascs)]
    return GridFront(cascades=cascs, evals=evals, config_index=idx_h, n_configs=sweep.n_configs)


# ------------------------------------------------------- device sampler --
class gs_sampler_job(ctypes.Structure):
    _fields_ = [("rng_state_hi", ctypes.c_uint64), ("rng_state_lo", ctypes.c_uint64),
                ("rng_inc_hi", ctypes.c_uint64), ("rng_inc_lo", ctypes.c_uint64),
                ("rng_has_uint32", ctypes.c_uint32), ("rng_uinteger", ctypes.c_uint32),
                ("n_samples", ctypes.c_int64), ("stage_model", ctypes.c_void_p),
                ("thresholds", ctypes.c_void_p), ("n_stages", ctypes.c_void_p),
                ("grid_index", ctypes.c_void_p), ("table", ctypes.c_void_p),
                ("table_cap", ctypes.c_int64), ("result", ctypes.c_void_p)]


@dataclass
class SampledCascades:
    """Device-resident output of sample_cascades_device for one seed:
    evaluate_encoded's encoding (model columns in profile order) plus each
    non-final stage's threshold index into its grid."""

    stage_model: torch.Tensor   # i32 [count, M], -1 padded
    thresholds: torch.Tensor    # f64 [count, M], 0 padded
    n_stages: torch.Tensor      # i32 [count]
    grid_index: torch.Tensor    # i32 [count, M], -1 padded
    count: int
    rng_state: tuple            # (state, has_uint32, uinteger) after sampling

    def cascades(self, model_ids) -> list[Cascade]:
        sm, th, ns = (t.cpu().numpy() for t in (self.stage_model, self.thresholds,
                                                 self.n_stages))
        return [Cascade(stages=tuple(model_ids[int(m)] for m in sm[i, :ns[i]]),
                        thresholds=tuple(float(x) for x in th[i, : ns[i] - 1]))
                for i in range(self.count)]


def sample_cascades_device(profiles: ProfileSet, grid: ThresholdGrid, n_samples: int,
                           rng_seeds) -> list[SampledCascades]:
    """sample_cascades (reference :166-193) on the device for one or many
    seeds in one launch (gs_sample_cascades): per seed, the same cascades in
    the same order as the host sampler, kept on the device in
    evaluate_encoded's encoding."""
    if n_samples < 1:
        raise ValueError(f"n_samples must be >= 1, got {n_samples}")
    seeds = [rng_seeds] if np.isscalar(rng_seeds) else list(rng_seeds)
    dev = _lib.device()
    ids = list(profiles.model_ids)
    M = len(ids)
    order = sorted(ids, key=lambda m: (profiles[m].runtime_table[1], profiles.index(m)))
    order_cols = np.array([profiles.index(m) for m in order], dtype=np.int32)
    vals, off = [], [0]
    for m in ids:
        g = grid.per_model[m]
        if len(g) >= 65536:
            raise ValueError("device sampler supports grids of < 65536 values")
        vals.extend(float(x) for x in g)
        off.append(len(vals))
    d_order = _lib.to_device(order_cols, torch.int32)
    d_grid = _lib.to_device(np.array(vals, dtype=np.float64), torch.float64)
    d_off = _lib.to_device(np.array(off, dtype=np.int32), torch.int32)
    cap = M + int(n_samples)
    tcap = 1 << max(4, int(2 * cap - 1).bit_length())
    outs, raw = [], b""
    for seed in seeds:
        st = np.random.default_rng(seed).bit_generator.state
        s, inc = int(st["state"]["state"]), int(st["state"]["inc"])
        o = {"sm": torch.empty((cap, M), dtype=torch.int32, device=dev),
             "th": torch.empty((cap, M), dtype=torch.float64, device=dev),
             "ns": torch.empty(cap, dtype=torch.int32, device=dev),
             "gi": torch.empty((cap, M), dtype=torch.int32, device=dev),
             "tab": torch.zeros(2 * tcap, dtype=torch.int64, device=dev),
             "res": torch.zeros(5, dtype=torch.int64, device=dev)}
        m64 = (1 << 64) - 1
        job = gs_sampler_job(s >> 64, s & m64, inc >> 64, inc & m64, int(st["has_uint32"]),
                             int(st["uinteger"]), int(n_samples), o["sm"].data_ptr(),
                             o["th"].data_ptr(), o["ns"].data_ptr(), o["gi"].data_ptr(),
                             o["tab"].data_ptr(), tcap, o["res"].data_ptr())
        raw += bytes(job)
        outs.append(o)
    table = torch.from_numpy(np.frombuffer(raw, dtype=np.uint8).copy()).to(dev)
    _lib.check(_lib.load().gs_sample_cascades(M, d_order.data_ptr(), d_grid.data_ptr(),
                                              d_off.data_ptr(), table.data_ptr(), len(seeds),
                                              _lib.stream_ptr()), "sample_cascades")
    res = torch.stack([o["res"] for o in outs]).cpu().numpy()
    out = []
    for o, r in zip(outs, res):
        n = int(r[0])
        state = (int(np.uint64(r[1])) << 64) | int(np.uint64(r[2]))
        out.append(SampledCascades(o["sm"][:n], o["th"][:n], o["ns"][:n], o["gi"][:n], n,
                                   (state, int(r[3]), int(r[4]))))
    return out
