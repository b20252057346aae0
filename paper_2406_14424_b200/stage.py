"""Online cascade stage step on the device.

Reference: EngineState.finish_batch (/root/reference/pkg/src/gearserve/
engine.py:355-383) — per item, in batch order: stop if the stage is the
gear's last or cert[row, m] >= thr (inclusive), else forward to the next
stage's queue — with certainty per cascades.certainty (src/cascades.py:20-28).

stage_step(): certainty of each row's scores (margin = Eq. 5, bit-exact;
max_softmax / entropy are extensions), the gate, order-preserving
compaction of the deferred rows, rows whose certainty is within near_eps of
their threshold listed, and the deferred rows' payload gathered contiguously
into the next stage's batch buffer — one kernel (csrc/gs_stage.cu).

stage_gate(): the same gate over the engine's precomputed certainty
matrices (CompiledPlan.cert/corr, src/engine.py:217), per item
(row, model, threshold, is_last), returning stop / correct / deferred order.
"""

from __future__ import annotations

import ctypes
import struct
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib

NEAR_EPS = 1e-6


@dataclass
class StageStepResult:
    cert: torch.Tensor            # f64 [n]
    stop: torch.Tensor            # u8 [n]
    deferred_idx: torch.Tensor    # i64 [n_deferred], batch order
    near_idx: torch.Tensor        # i64 [n_near], ascending
    next_payload: torch.Tensor | None  # [n_deferred, ...] gathered payload rows
    counts: torch.Tensor | None = None  # device i64 [2]: n_deferred, n_near


def _thr_tensor(thr, n: int, dev) -> torch.Tensor:
    if isinstance(thr, (int, float)):
        return torch.full((n,), float(thr), dtype=torch.float64, device=dev)
    t = _lib.to_device(thr, torch.float64)
    if t.numel() != n:
        raise ValueError("thr must be a scalar or one threshold per row")
    return t


def stage_step(scores: torch.Tensor, thr, is_last=None, *, kind: str = "margin",
               payload: torch.Tensor | None = None, near_eps: float = NEAR_EPS,
               list_near: bool = True, sync: bool = True) -> StageStepResult:
    """Gate one stage's batch.  scores: CUDA [n, n_cls] f32/f64/bf16 (row
    stride may exceed n_cls); thr: scalar or [n] f64; is_last: None or [n]
    bool/u8; payload: optional CUDA tensor with leading dim n.  With
    sync=False nothing is read back: deferred_idx / near_idx are returned at
    full capacity and `counts` (device i64 [2]: n_deferred, n_near) says how
    much of each is valid."""
    if kind not in _lib.CERT_KINDS:
        raise ValueError(f"unknown certainty kind {kind!r}")
    dev = _lib.device()
    if scores.device.type != "cuda":
        scores = _lib.to_device(scores, scores.dtype)
    if scores.dtype not in _lib.DTYPES:
        raise ValueError(f"unsupported score dtype {scores.dtype}")
    if scores.ndim != 2 or scores.stride(1) != 1:
        raise ValueError("scores must be a row-major [n_rows, n_cls] matrix")
    n, c = int(scores.shape[0]), int(scores.shape[1])
    if c == 0:
        raise ValueError("certainty of empty scores")
    th = _thr_tensor(thr, n, dev)
    last = None
    if is_last is not None:
        last = _lib.to_device(is_last, torch.uint8) if not isinstance(is_last, torch.Tensor) \
            else is_last.to(dev, torch.uint8).contiguous()
        if last.numel() != n:
            raise ValueError("is_last must have one flag per row")
    cert = torch.empty(n, dtype=torch.float64, device=dev)
    stop = torch.empty(n, dtype=torch.uint8, device=dev)
    deferred = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
    near = torch.empty(max(n, 1), dtype=torch.int64, device=dev) if list_near else None
    counts = torch.zeros(2, dtype=torch.int64, device=dev)
    nxt = None
    row_bytes = 0
    if payload is not None:
        if payload.shape[0] != n or not payload.is_contiguous() or payload.device.type != "cuda":
            raise ValueError("payload must be a contiguous CUDA tensor with one row per score row")
        row_bytes = payload[0].numel() * payload.element_size() if n else 0
        nxt = torch.empty_like(payload)
    lib = _lib.load()
    nbytes = ctypes.c_size_t()
    _lib.check(lib.gs_stage_step_workspace(n, ctypes.byref(nbytes)), "stage_step")
    ws = _lib.workspace(nbytes.value)
    rc = lib.gs_stage_step(
        scores.data_ptr() if n else None, _lib.DTYPES[scores.dtype], n, c, _lib.row_stride(scores),
        _lib.CERT_KINDS[kind], th.data_ptr() if n else None, _lib.ptr(last),
        cert.data_ptr(), stop.data_ptr(), deferred.data_ptr(), counts.data_ptr(),
        float(near_eps), _lib.ptr(near), counts.data_ptr() + 8 if list_near else None,
        _lib.ptr(payload), row_bytes, _lib.ptr(nxt), ws.data_ptr(), ws.numel(),
        _lib.stream_ptr())
    _lib.check(rc, "stage_step")
    if not sync:
        return StageStepResult(cert=cert, stop=stop, deferred_idx=deferred,
                               near_idx=near if list_near else deferred[:0],
                               next_payload=nxt, counts=counts)
    nd, nn = (int(x) for x in counts.tolist())
    return StageStepResult(cert=cert, stop=stop, deferred_idx=deferred[:nd],
                           near_idx=near[:nn] if list_near else deferred[:0],
                           next_payload=None if nxt is None else nxt[:nd], counts=counts)


@dataclass
class GateResult:
    stop: torch.Tensor           # u8 [n_items]
    correct: torch.Tensor        # u8 [n_items] (0 for forwarded items)
    deferred_idx: torch.Tensor   # i64 item positions, batch order
    near_idx: torch.Tensor       # i64 item positions within near_eps


def stage_gate(cert: torch.Tensor, corr: torch.Tensor, row, model, thr, is_last=None, *,
               near_eps: float = NEAR_EPS) -> GateResult:
    """Gate items against precomputed certainty/correct matrices."""
    dev = _lib.device()
    rows = _lib.to_device(row, torch.int64)
    models = _lib.to_device(model, torch.int32)
    n = int(rows.numel())
    th = _thr_tensor(thr, n, dev)
    last = None if is_last is None else _lib.to_device(
        np.asarray(is_last, dtype=np.uint8) if not isinstance(is_last, torch.Tensor) else is_last,
        torch.uint8)
    stop = torch.empty(n, dtype=torch.uint8, device=dev)
    correct = torch.empty(n, dtype=torch.uint8, device=dev)
    deferred = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
    near = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
    counts = torch.zeros(2, dtype=torch.int64, device=dev)
    lib = _lib.load()
    nbytes = ctypes.c_size_t()
    _lib.check(lib.gs_stage_step_workspace(n, ctypes.byref(nbytes)), "stage_gate")
    ws = _lib.workspace(nbytes.value)
    rc = lib.gs_stage_gate(cert.data_ptr(), corr.data_ptr(), int(cert.shape[0]),
                           int(cert.shape[1]), rows.data_ptr() if n else None,
                           models.data_ptr() if n else None, th.data_ptr() if n else None,
                           _lib.ptr(last), n, stop.data_ptr(), correct.data_ptr(),
                           deferred.data_ptr(), counts.data_ptr(), float(near_eps),
                           near.data_ptr(), counts.data_ptr() + 8, ws.data_ptr(), ws.numel(),
                           _lib.stream_ptr())
    _lib.check(rc, "stage_gate")
    nd, nn = (int(x) for x in counts.tolist())
    return GateResult(stop=stop, correct=correct, deferred_idx=deferred[:nd],
                      near_idx=near[:nn])


class GateBatcher:
    """The gate for small online batches as ONE native call per batch
    (gs_stage_gate_packed): the items go to the device in one pinned H2D,
    the outcome comes back in one pinned D2H, buffers reused across calls.

    The reference gates a batch of <= max_profiled_batch items (4-8,
    src/synth.py:30) per finish_batch (src/engine.py:355-383); at that size
    a gate is latency-bound, so what matters is the number of host<->device
    transfers and launches per batch: one copy in, one kernel, one copy out.
    """

    def __init__(self, cert: torch.Tensor, corr: torch.Tensor, capacity: int = 64,
                 near_eps: float = NEAR_EPS):
        self.cert = _lib.to_device(cert, torch.float64)
        self.corr = _lib.to_device(corr, torch.uint8)
        if self.cert.ndim != 2 or tuple(self.corr.shape) != tuple(self.cert.shape):
            raise ValueError("cert and corr must both be [n_records, n_models]")
        self.n_rec, self.n_models = int(self.cert.shape[0]), int(self.cert.shape[1])
        self.near_eps = float(near_eps)
        self.cap = 0
        self._args = None
        self._args_cap = 0
        self._graphs: dict = {}  # n -> captured packed-gate graph (gate_small)
        self._grow(max(1, int(capacity)))

    def _grow(self, n: int) -> None:
        lib = _lib.load()
        hin, hout, dev = ctypes.c_size_t(), ctypes.c_size_t(), ctypes.c_size_t()
        _lib.check(lib.gs_stage_gate_packed_bytes(n, ctypes.byref(hin), ctypes.byref(hout),
                                                  ctypes.byref(dev)), "gate batch")
        self.h_in = torch.empty(max(hin.value, 8), dtype=torch.uint8, pin_memory=True)
        self.h_out = torch.empty(max(hout.value, 16), dtype=torch.uint8, pin_memory=True)
        self.d_buf = _lib.workspace(dev.value)
        self._in = self.h_in.numpy()
        self._out = self.h_out.numpy()
        self.cap = n

    def gate_small(self, rows: list, model: list, thr: list, is_last: list):
        """gate() for a handful of items given as Python lists (the online
        batch of finish_batch): struct packing into the pinned buffer, the
        same single C call, the outcome as Python lists (stop, correct,
        near positions)."""
        n = len(rows)
        if n > self.cap:
            self._grow(max(n, 2 * self.cap))
        if self._args is None or self._args_cap != self.cap:
            self._lib = _lib.load()
            self._mv_in = memoryview(self._in)
            self._mv_out = memoryview(self._out)
            self._args = (self.cert.data_ptr(), self.corr.data_ptr(), self.n_rec, self.n_models,
                          self.h_in.data_ptr())
            self._args2 = (self.near_eps, self.h_out.data_ptr(), self.d_buf.data_ptr(), self.d_buf.numel(), 1)
            self._args_cap = self.cap
            self._graphs = {}
        struct.pack_into(f"<{n}q{n}d{n}i{n}?", self._mv_in, 0, *rows, *thr, *model, *is_last)
        if n in self._graphs:
            graph = self._graphs[n]  # None: capture failed here once, use the plain call
        else:
            graph = self._capture(n) if len(self._graphs) < 64 else None
        if graph is not None:  # H2D, gate, D2H as one graph launch
            graph.replay()
            torch.cuda.current_stream().synchronize()
        else:
            rc = self._lib.gs_stage_gate_packed(*self._args, n, *self._args2, _lib.stream_ptr())
            _lib.check(rc, "gate batch")
        n_near = struct.unpack_from("<q", self._mv_out, 8)[0]
        flags = struct.unpack_from(f"<{2 * n}B", self._mv_out, 16)
        near = struct.unpack_from(f"<{n_near}q", self._mv_out, (16 + 2 * n + 7) // 8 * 8) if n_near else ()
        return flags[:n], flags[n:], near

    def _capture(self, n: int):
        """The packed gate call for n items as a CUDA graph (its buffers are
        fixed), or None when capture is not possible here."""
        try:
            rc = self._lib.gs_stage_gate_packed(*self._args, n, *self._args2, _lib.stream_ptr())  # warm
            _lib.check(rc, "gate batch")
            g = torch.cuda.CUDAGraph()
            a2 = self._args2[:-1] + (0,)  # no synchronize inside the graph
            with torch.cuda.graph(g):
                rc = self._lib.gs_stage_gate_packed(*self._args, n, *a2, _lib.stream_ptr())
            _lib.check(rc, "gate batch")
        except RuntimeError:
            self._graphs[n] = None
            return None
        self._graphs[n] = g
        return g

    def gate(self, rows, model, thr, is_last):
        """(stop bool[n], correct u8[n], near positions i64) for one batch;
        rows i64, model i32, thr f64, is_last bool — host arrays."""
        n = len(rows)
        if n > self.cap:
            self._grow(max(n, 2 * self.cap))
        b = self._in
        b[: 8 * n].view(np.int64)[:] = rows
        b[8 * n: 16 * n].view(np.float64)[:] = thr
        b[16 * n: 20 * n].view(np.int32)[:] = model
        b[20 * n: 21 * n] = is_last
        rc = _lib.load().gs_stage_gate_packed(
            self.cert.data_ptr(), self.corr.data_ptr(), self.n_rec, self.n_models,
            self.h_in.data_ptr(), n, self.near_eps, self.h_out.data_ptr(), self.d_buf.data_ptr(),
            self.d_buf.numel(), 1, _lib.stream_ptr())
        _lib.check(rc, "gate batch")
        o = self._out
        n_near = int(o[8:16].view(np.int64)[0])
        stop = o[16: 16 + n].astype(bool)
        correct = o[16 + n: 16 + 2 * n].copy()
        near_off = (16 + 2 * n + 7) // 8 * 8
        near = o[near_off: near_off + 8 * n_near].view(np.int64).copy()
        return stop, correct, near
