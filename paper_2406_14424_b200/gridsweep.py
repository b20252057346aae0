"""Full-grid gear-plan sweep over a validation set resident in HBM.

Scores every (cascade structure x per-stage threshold) config of the grid
product — the search space planner SP1 samples from
(/root/reference/pkg/src/gearserve/planner.py:365-390 via
cascades.sample_cascades, src/cascades.py:166-193) — with the reference's
per-config outputs (accuracy, mean_cost, forward_frac; src/kernels.py:39-62)
and the reference's Pareto semantics (src/cascades.py:116-129).

Config enumeration (identical in the kernels, here, and in oracle/):
structures are the non-empty model subsets in column order (columns are the
cost order), by size then lexicographically (itertools.combinations); a
structure (m_1..m_K) owns prod_{s<K} |grid[m_s]| configs whose threshold
indices (k_1..k_{K-1}) are lexicographic with k_1 slowest.  Config c decodes
to the encoded cascade stage_model = (m_1..m_K, -1 pad),
thresholds = (grid[m_1][k_1], ..., grid[m_{K-1}][k_{K-1}], 0 pad).
"""

from __future__ import annotations

import ctypes
import itertools
from dataclasses import dataclass
from typing import Sequence

import numpy as np
import torch

from . import _lib
from .types import Cascade

GS_GRID_WORKSPACE_DIRTY = 1
GS_GRID_BUILD_RECORDS_PASS = 2
GS_GRID_BUILD_TABLES_PASS = 4


def structures(n_models: int, grid_len: Sequence[int]) -> list[tuple[tuple[int, ...], int, int]]:
    """[(models, first_config, n_configs)] in enumeration order."""
    out = []
    off = 0
    for k in range(1, n_models + 1):
        for combo in itertools.combinations(range(n_models), k):
            n = 1
            for m in combo[:-1]:
                n *= int(grid_len[m])
            out.append((combo, off, n))
            off += n
    return out


def n_configs(grid_len: Sequence[int]) -> int:
    return sum(n for _, _, n in structures(len(grid_len), grid_len))


@dataclass
class SweepResult:
    accuracy: torch.Tensor | None
    mean_cost: torch.Tensor | None
    forward_frac: torch.Tensor | None
    n_correct: torch.Tensor | None
    config_begin: int


class GridSweep:
    """Histogram + prefix tables for one validation set and one grid,
    built once (gs_grid_build); configs are then scored in ranges
    (gs_grid_eval) and reduced to a Pareto front (gs_pareto_counts)."""

    def __init__(self, certainty, correct, grids: Sequence, cost1, *, build: bool = True):
        dev = _lib.device()
        self.cert = _lib.to_device(certainty, torch.float64)
        self.corr = _lib.to_device(correct, torch.uint8)
        if self.cert.ndim != 2 or tuple(self.corr.shape) != tuple(self.cert.shape):
            raise ValueError("certainty and correct must both be [n_records, n_models]")
        self.n_rec, self.n_models = int(self.cert.shape[0]), int(self.cert.shape[1])
        if len(grids) != self.n_models:
            raise ValueError(f"need {self.n_models} grids, got {len(grids)}")
        host_grids = []
        for j, g in enumerate(grids):
            g = np.asarray(g.cpu() if isinstance(g, torch.Tensor) else g, dtype=np.float64)
            if g.ndim != 1 or g.size == 0:
                raise ValueError(f"grid {j} must be a non-empty 1-D array")
            if np.any(np.diff(g) <= 0):
                raise ValueError(f"grid {j} is not strictly increasing")
            host_grids.append(g)
        self.grids_host = host_grids
        self.grid_len = [int(g.size) for g in host_grids]
        self._glen = _lib.int32_array(self.grid_len)
        self.grids = _lib.to_device(np.concatenate(host_grids), torch.float64)
        self.cost1 = _lib.to_device(np.asarray(cost1, dtype=np.float64), torch.float64)
        if self.cost1.numel() != self.n_models:
            raise ValueError("cost1 must have one entry per model")
        info = _lib.gs_grid_info()
        lib = _lib.load()
        _lib.check(lib.gs_grid_plan(self.n_rec, self.n_models, self._glen, ctypes.byref(info)),
                   "grid plan")
        self.info = info
        self.n_configs = int(info.n_configs)
        self.max_len = int(info.max_len)
        # zeroed once: each build leaves its histogram region zero again
        self.table = torch.zeros(int(info.workspace_bytes), dtype=torch.uint8, device=dev)
        self._built = False
        self._clean = True
        if build:
            self.build()

    # -- table -------------------------------------------------------------
    def build(self, part: str | None = None) -> None:
        """Fill the prefix tables from the device matrices.  part = "records"
        / "tables" runs one of the build's two passes (four-model path; for
        timing them apart), "records" first."""
        lib = _lib.load()
        flags = 0 if self._clean else GS_GRID_WORKSPACE_DIRTY
        if part == "records":
            flags |= GS_GRID_BUILD_RECORDS_PASS
        elif part == "tables":
            flags = GS_GRID_BUILD_TABLES_PASS
        elif part is not None:
            raise ValueError(f"unknown build part {part!r}")
        rc = lib.gs_grid_build(self.cert.data_ptr(), self.corr.data_ptr(), self.n_rec,
                               self.n_models, self.grids.data_ptr(), self._glen,
                               self.table.data_ptr(), self.table.numel(), flags,
                               _lib.stream_ptr())
        if rc != _lib.GS_OK:
            self._clean = False
        _lib.check(rc, "grid build")
        self._clean = part != "records"
        self._built = part != "records"

    def build_streamed(self, certainty_host: torch.Tensor, correct_host: torch.Tensor,
                       chunks: int = 8) -> None:
        """Build from HOST matrices (pinned torch tensors of this sweep's
        shape), overlapping the host->device copy of each record slice with
        the binning of the previous ones (gs_grid_accumulate per slice on the
        current stream, copies on a side stream, then gs_grid_finish).  The
        copies land in this sweep's device matrices.  Four-model fast path
        only (gs_grid_info.fast_path)."""
        if not self.info.fast_path:
            raise ValueError("streamed build needs the four-model fast path "
                             "(gs_grid_info.fast_path == 0 for this shape)")
        if (tuple(certainty_host.shape) != tuple(self.cert.shape)
                or tuple(correct_host.shape) != tuple(self.corr.shape)
                or certainty_host.dtype != torch.float64 or correct_host.dtype != torch.uint8):
            raise ValueError("host matrices must match the sweep's [n_rec, n_models] f64 / u8")
        lib = _lib.load()
        main = torch.cuda.current_stream()
        if getattr(self, "_copy_stream", None) is None:
            self._copy_stream = torch.cuda.Stream()
        copy = self._copy_stream
        copy.wait_stream(main)  # earlier work on the device matrices is done
        flags = 0 if self._clean else GS_GRID_WORKSPACE_DIRTY
        bounds = np.linspace(0, self.n_rec, max(1, int(chunks)) + 1).astype(np.int64)
        for lo, hi in zip(bounds[:-1], bounds[1:]):
            lo, hi = int(lo), int(hi)
            if hi <= lo:
                continue
            with torch.cuda.stream(copy):
                self.cert[lo:hi].copy_(certainty_host[lo:hi], non_blocking=True)
                self.corr[lo:hi].copy_(correct_host[lo:hi], non_blocking=True)
                done = torch.cuda.Event()
                done.record(copy)
            main.wait_event(done)
            rc = lib.gs_grid_accumulate(self.cert[lo:].data_ptr(), self.corr[lo:].data_ptr(),
                                        hi - lo, self.n_rec, self.n_models,
                                        self.grids.data_ptr(), self._glen,
                                        self.table.data_ptr(), self.table.numel(), flags,
                                        main.cuda_stream)
            _lib.check(rc, "grid accumulate")
            flags = 0
        self._clean = False  # the histogram holds records until finish
        rc = lib.gs_grid_finish(self.n_rec, self.n_models, self._glen, self.table.data_ptr(),
                                self.table.numel(), main.cuda_stream)
        _lib.check(rc, "grid finish")
        self._clean = True
        self._built = True

    # -- scoring -----------------------------------------------------------
    def evaluate(self, begin: int = 0, count: int | None = None, *, accuracy: bool = True,
                 mean_cost: bool = True, forward_frac: bool = True,
                 n_correct: bool = False, out: SweepResult | None = None) -> SweepResult:
        if not self._built:
            raise RuntimeError("GridSweep.build() has not run")
        if count is None:
            count = self.n_configs - begin
        if begin < 0 or count < 0 or begin + count > self.n_configs:
            raise ValueError("config range outside the enumeration")
        dev = self.cert.device
        if out is None:
            f64 = dict(dtype=torch.float64, device=dev)
            out = SweepResult(
                torch.empty(count, **f64) if accuracy else None,
                torch.empty(count, **f64) if mean_cost else None,
                torch.empty((count, self.max_len), **f64) if forward_frac else None,
                torch.empty(count, dtype=torch.int32, device=dev) if n_correct else None,
                begin)
        else:
            _check_out(out, count, self.max_len, dev)
        out.config_begin = begin
        lib = _lib.load()
        rc = lib.gs_grid_eval(self.n_rec, self.n_models, self._glen, self.cost1.data_ptr(),
                              begin, count, _lib.ptr(out.accuracy), _lib.ptr(out.mean_cost),
                              _lib.ptr(out.forward_frac), _lib.ptr(out.n_correct),
                              self.table.data_ptr(), self.table.numel(), _lib.stream_ptr())
        _lib.check(rc, "grid eval")
        return out

    def histogram(self) -> None:
        """The histogram half of build() (fast path): gs_grid_accumulate over
        all records.  Leaves the workspace mid-build until finish()."""
        lib = _lib.load()
        flags = 0 if self._clean else GS_GRID_WORKSPACE_DIRTY
        rc = lib.gs_grid_accumulate(self.cert.data_ptr(), self.corr.data_ptr(), self.n_rec,
                                    self.n_rec, self.n_models, self.grids.data_ptr(), self._glen,
                                    self.table.data_ptr(), self.table.numel(), flags,
                                    _lib.stream_ptr())
        _lib.check(rc, "grid accumulate")
        self._clean = False

    def finish(self) -> None:
        """The prefix-table half of build() (fast path): gs_grid_finish."""
        lib = _lib.load()
        rc = lib.gs_grid_finish(self.n_rec, self.n_models, self._glen, self.table.data_ptr(),
                                self.table.numel(), _lib.stream_ptr())
        _lib.check(rc, "grid finish")
        self._clean = True
        self._built = True

    def capture(self, out: SweepResult, build: bool = True, evaluate: bool = True,
                part: str | None = None) -> torch.cuda.CUDAGraph:
        """CUDA graph of one sweep step (table build and/or scoring every
        config into `out`), so a step is one graph launch instead of a
        Python-driven sequence of kernel launches.  part = "records" /
        "tables" captures one pass of the build alone (for timing)."""
        def body():
            if part in ("records", "tables"):
                self.build(part=part)
                return
            if build:
                self.build()
            if evaluate:
                self.evaluate(out=out)
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            body()  # first call does one-time kernel attribute setup outside capture
        torch.cuda.current_stream().wait_stream(side)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            body()
        return graph

    def pareto(self, begin: int = 0, count: int | None = None,
               res: SweepResult | None = None) -> tuple[torch.Tensor, SweepResult]:
        """Config indices (ascending) of the Pareto front of [begin, begin+count),
        plus the scored range."""
        if res is None:
            res = self.evaluate(begin, count, accuracy=True, mean_cost=True,
                                forward_frac=True, n_correct=True)
        elif res.n_correct is None or res.mean_cost is None:
            raise ValueError("pareto(res=...) needs a result scored with n_correct=True "
                             "and mean_cost")
        idx = pareto_counts(res.n_correct, res.mean_cost, self.n_rec, base_index=res.config_begin)
        return idx, res

    # -- decoding ----------------------------------------------------------
    def decode(self, config_idx) -> tuple[torch.Tensor, torch.Tensor, torch.Tensor]:
        idx = _lib.to_device(config_idx, torch.int64)
        n = int(idx.numel())
        dev = self.cert.device
        sm = torch.empty((n, self.n_models), dtype=torch.int32, device=dev)
        thr = torch.empty((n, self.n_models), dtype=torch.float64, device=dev)
        ns = torch.empty(n, dtype=torch.int32, device=dev)
        if n:
            if int(idx.min()) < 0 or int(idx.max()) >= self.n_configs:
                raise IndexError("config index outside the enumeration")
            lib = _lib.load()
            rc = lib.gs_grid_decode(self.n_models, self._glen, self.grids.data_ptr(),
                                    idx.data_ptr(), n, sm.data_ptr(), thr.data_ptr(),
                                    ns.data_ptr(), _lib.stream_ptr())
            _lib.check(rc, "grid decode")
        return sm, thr, ns

    def cascades(self, config_idx, model_ids: Sequence[str]) -> list[Cascade]:
        sm, thr, ns = (t.cpu().numpy() for t in self.decode(config_idx))
        out = []
        for i in range(sm.shape[0]):
            k = int(ns[i])
            out.append(Cascade(stages=tuple(model_ids[int(m)] for m in sm[i, :k]),
                               thresholds=tuple(float(x) for x in thr[i, :k - 1])))
        return out


def _check_out(out: SweepResult, count: int, max_len: int, dev: torch.device) -> None:
    """A caller-supplied SweepResult must hold `count` configs in the layout
    gs_grid_eval writes (the C call receives no output sizes)."""
    specs = (("accuracy", out.accuracy, torch.float64, (count,)),
             ("mean_cost", out.mean_cost, torch.float64, (count,)),
             ("forward_frac", out.forward_frac, torch.float64, (count, max_len)),
             ("n_correct", out.n_correct, torch.int32, (count,)))
    for name, t, dtype, shape in specs:
        if t is None:
            continue
        if t.dtype != dtype or t.device != dev or not t.is_contiguous():
            raise ValueError(f"out.{name} must be a contiguous {dtype} tensor on {dev}")
        if tuple(t.shape) != shape:
            raise ValueError(f"out.{name} has shape {tuple(t.shape)}, the range needs {shape}")


def front_rows(idx: torch.Tensor, res: SweepResult) -> torch.Tensor:
    """Device [n_front, 3 + max_len] f64 rows (config index, accuracy,
    mean_cost, forward_frac...) of the configs `idx` (absolute indices) of a
    scored range, so a front leaves the device in one copy."""
    local = idx - res.config_begin
    cols = [idx.to(torch.float64)[:, None], res.accuracy[local][:, None],
            res.mean_cost[local][:, None], res.forward_frac[local]]
    return torch.cat(cols, dim=1)


def front_host(idx: torch.Tensor, res: SweepResult) -> np.ndarray:
    """front_rows copied to host memory in one pinned D2H: [n_front, 3 +
    max_len] f64 (config index, accuracy, mean_cost, forward_frac...)."""
    rows = front_rows(idx, res)
    host = _pinned(rows.shape, rows.dtype)
    host.copy_(rows, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    return host.numpy().copy()  # the pinned staging buffer is reused by the next call


_PINNED: dict = {}


def _pinned(shape, dtype) -> torch.Tensor:
    """A pinned host buffer of at least `shape`, reused across calls (one
    per dtype, grown geometrically)."""
    n = int(np.prod(shape))
    buf = _PINNED.get(dtype)
    if buf is None or buf.numel() < n:
        buf = torch.empty(max(n, 1 << 16) * 2, dtype=dtype, pin_memory=True)
        _PINNED[dtype] = buf
    return buf[:n].view(*shape)


class _ParetoScratch:
    """Workspace, outputs and a pinned count slot of gs_pareto_counts for one
    (n, n_rec, device), allocated once and reused."""

    def __init__(self, n: int, n_rec: int, dev: torch.device):
        lib = _lib.load()
        nbytes = ctypes.c_size_t()
        _lib.check(lib.gs_pareto_counts_workspace(n, n_rec, ctypes.byref(nbytes)), "pareto")
        self.ws = _lib.workspace(nbytes.value)
        self.kept = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
        self.n_kept = torch.zeros(1, dtype=torch.int64, device=dev)
        self.n_host = torch.zeros(1, dtype=torch.int64, pin_memory=True)


_SCRATCH: dict = {}


def pareto_counts(n_correct: torch.Tensor, mean_cost: torch.Tensor, n_rec: int,
                  base_index: int = 0, keep: torch.Tensor | None = None) -> torch.Tensor:
    """Indices (+base_index, ascending) of the exact Pareto front of points
    given as integer correct counts and f64 costs (gs_pareto_counts).
    Workspace and outputs are reused across calls of the same shape."""
    lib = _lib.load()
    n = int(n_correct.numel())
    dev = _lib.device()
    key = (n, int(n_rec), dev.index)
    sc = _SCRATCH.get(key)
    if sc is None:
        if len(_SCRATCH) > 8:
            _SCRATCH.clear()
        sc = _SCRATCH[key] = _ParetoScratch(n, n_rec, dev)
    rc = lib.gs_pareto_counts(n_correct.data_ptr() if n else None,
                              mean_cost.data_ptr() if n else None, n, n_rec, base_index,
                              _lib.ptr(keep), sc.kept.data_ptr(), sc.n_kept.data_ptr(),
                              sc.ws.data_ptr(), sc.ws.numel(), _lib.stream_ptr())
    _lib.check(rc, "pareto")
    sc.n_host.copy_(sc.n_kept, non_blocking=True)
    torch.cuda.current_stream().synchronize()
    return sc.kept[: int(sc.n_host[0])].clone()


class BatchedSweep:
    """Full grid sweeps of many validation sets of M models: certainty
    [R, n, M] f64, correct [R, n, M] u8, grids [R][M] per-set grids (each
    strictly increasing; the M lengths shared by every set), cost1 [M].
    run() fills [R, C] accuracy / mean_cost and [R, C, M] forward_frac, each
    row equal to that set's GridSweep(...).evaluate().  Three models (config
    1 stacked: the reference's CPU default is launch-bound as one sweep) take
    one launch per run() (gs_grid_sweep_batched); other M run the sets'
    sweeps back to back on the stream (one workspace per set, built here).
    The constructor does the host work (validation, grid upload)."""

    def __init__(self, certainty, correct, grids, cost1):
        self.cert = _lib.to_device(certainty, torch.float64)
        self.corr = _lib.to_device(correct, torch.uint8)
        if (self.cert.ndim != 3 or tuple(self.corr.shape) != tuple(self.cert.shape)
                or self.cert.shape[2] < 1):
            raise ValueError("certainty and correct must both be [n_sets, n_records, n_models]")
        self.n_sets, self.n_rec = int(self.cert.shape[0]), int(self.cert.shape[1])
        M = self.n_models = int(self.cert.shape[2])
        if len(grids) != self.n_sets:
            raise ValueError(f"need {self.n_sets} grid sets, got {len(grids)}")
        glen = None
        flat = []
        for s_idx, triple in enumerate(grids):
            if len(triple) != M:
                raise ValueError(f"set {s_idx}: need {M} grids")
            lens = []
            for j, g in enumerate(triple):
                g = np.asarray(g.cpu() if isinstance(g, torch.Tensor) else g, dtype=np.float64)
                if g.ndim != 1 or g.size == 0 or np.any(np.diff(g) <= 0):
                    raise ValueError(f"set {s_idx} grid {j} must be a non-empty strictly "
                                     "increasing 1-D array")
                lens.append(int(g.size))
                flat.append(g)
            if glen is None:
                glen = lens
            elif lens != glen:
                raise ValueError("every set's grids must have the same lengths")
        self.grid_len = glen
        self._glen = _lib.int32_array(glen)
        self.grids = _lib.to_device(np.concatenate(flat), torch.float64)
        self.cost1 = _lib.to_device(np.asarray(cost1, dtype=np.float64), torch.float64)
        if self.cost1.numel() != M:
            raise ValueError(f"cost1 must have {M} entries")
        self._sweeps = None
        self._bufs = None
        if M == 3:
            g0, g1, _ = glen
            self.n_configs = 3 + 2 * g0 + g1 + g0 * g1
        else:  # one GridSweep per set (its own workspace), run back to back
            c1 = np.asarray(cost1, dtype=np.float64)
            self._sweeps = [GridSweep(self.cert[s], self.corr[s], list(grids[s]), c1, build=False)
                            for s in range(self.n_sets)]
            self.n_configs = self._sweeps[0].n_configs if self._sweeps else 0
        dev = self.cert.device
        self.out = SweepResult(
            accuracy=torch.empty((self.n_sets, self.n_configs), dtype=torch.float64, device=dev),
            mean_cost=torch.empty((self.n_sets, self.n_configs), dtype=torch.float64, device=dev),
            forward_frac=torch.empty((self.n_sets, self.n_configs, M), dtype=torch.float64,
                                     device=dev),
            n_correct=None, config_begin=0)

    def run(self) -> SweepResult:
        o = self.out
        if self._sweeps is not None:
            # each set scores into its sweep's own (aligned) buffers, then its
            # row of the stacked result (rows of an odd C are not 16-byte
            # aligned, which the vector stores need)
            if self._bufs is None:
                self._bufs = [None] * self.n_sets
            for s, sw in enumerate(self._sweeps):
                sw.build()
                self._bufs[s] = sw.evaluate(out=self._bufs[s])
                o.accuracy[s].copy_(self._bufs[s].accuracy)
                o.mean_cost[s].copy_(self._bufs[s].mean_cost)
                o.forward_frac[s].copy_(self._bufs[s].forward_frac)
            return o
        rc = _lib.load().gs_grid_sweep_batched(
            self.cert.data_ptr(), self.corr.data_ptr(), self.n_sets, self.n_rec, 3,
            self.grids.data_ptr(), self._glen, self.cost1.data_ptr(), o.accuracy.data_ptr(),
            o.mean_cost.data_ptr(), o.forward_frac.data_ptr(), _lib.stream_ptr())
        _lib.check(rc, "batched grid sweep")
        return o


def sweep_batched(certainty, correct, grids, cost1) -> SweepResult:
    """BatchedSweep(...).run(): every set's full sweep in one launch."""
    return BatchedSweep(certainty, correct, grids, cost1).run()
