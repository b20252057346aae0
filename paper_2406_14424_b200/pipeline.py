"""Pipelined sweeps of host-resident validation sets.

A planner that re-sweeps as new validation data arrives (or sweeps many
tenants' sets with one grid shape) is bound by the host->device copy of the
certainty/correct matrices (36 MB per 1M x 4 set: ~0.7 ms over PCIe Gen5),
while the device work of a sweep (histogram, tables, every config, exact
Pareto front) takes well under 0.1 ms.  ``SweepPipeline`` keeps two device
slots: the copy of set i+1 runs on a copy stream while set i is swept, its
front reduced and read back, so the steady-state cost of a sweep approaches
the copy alone.  Results are the same rows ``gridsweep.front_host`` returns
for a single sweep (config index, accuracy, mean_cost, forward_frac...).

Stream/event protocol per slot s (two slots, alternating):
  copy stream:    wait(tail_done[s]) -> H2D into slot s -> record(h2d[s])
  compute stream: wait(h2d[s]) -> build, eval, Pareto kernels -> D2H of the
                  front size into pinned memory -> record(count[s])
  tail stream:    (after the host reads the size) wait(count[s]) -> gather
                  the front rows -> D2H into pinned memory -> record(tail_done[s])
The host only ever waits on a slot's count event while the other slot's
copy is already queued, so the copy engine never idles.
"""

from __future__ import annotations

import ctypes
from collections import deque
from typing import Sequence

import numpy as np
import torch

from . import _lib
from .gridsweep import GridSweep, _ParetoScratch, front_rows


class SweepPipeline:
    def __init__(self, n_rec: int, n_models: int, grids: Sequence, cost1, depth: int = 2):
        dev = _lib.device()
        self.n_rec, self.n_models = int(n_rec), int(n_models)
        self.depth = int(depth)
        self.slots = []
        for _ in range(self.depth):
            cert = torch.empty((n_rec, n_models), dtype=torch.float64, device=dev)
            corr = torch.empty((n_rec, n_models), dtype=torch.uint8, device=dev)
            sw = GridSweep(cert, corr, grids, cost1, build=False)
            self.slots.append({
                "sweep": sw, "cert": cert, "corr": corr, "out": None,
                "scratch": _ParetoScratch(sw.n_configs, n_rec, dev),
                "h2d": torch.cuda.Event(), "count": torch.cuda.Event(),
                "tail": torch.cuda.Event(), "used": False,
            })
        self.copy = torch.cuda.Stream()
        self.compute = torch.cuda.Stream()
        self.tail = torch.cuda.Stream()
        self.n_configs = self.slots[0]["sweep"].n_configs
        self._pending: deque = deque()  # (slot index, ticket)
        self._next = 0
        self._ticket = 0
        self._done: dict = {}

    def submit(self, certainty: torch.Tensor, correct: torch.Tensor) -> int:
        """Queue a sweep of pinned host matrices [n_rec, n_models] (f64 / u8);
        returns a ticket for result().  Blocks only when both slots are busy
        (then it finishes the oldest sweep first)."""
        if tuple(certainty.shape) != (self.n_rec, self.n_models) or \
                tuple(correct.shape) != (self.n_rec, self.n_models):
            raise ValueError("host matrices must be [n_rec, n_models]")
        if len(self._pending) >= self.depth:
            self._finish_oldest()
        s = self._next
        self._next = (self._next + 1) % self.depth
        slot = self.slots[s]
        lib = _lib.load()
        with torch.cuda.stream(self.copy):
            if slot["used"]:
                self.copy.wait_event(slot["tail"])  # the slot's last front has left
            slot["cert"].copy_(certainty, non_blocking=True)
            slot["corr"].copy_(correct, non_blocking=True)
            slot["h2d"].record(self.copy)
        slot["used"] = True
        with torch.cuda.stream(self.compute):
            self.compute.wait_event(slot["h2d"])
            sw = slot["sweep"]
            sw.build()
            slot["out"] = sw.evaluate(n_correct=True, out=slot["out"])
            sc = slot["scratch"]
            rc = lib.gs_pareto_counts(slot["out"].n_correct.data_ptr(),
                                      slot["out"].mean_cost.data_ptr(), self.n_configs,
                                      self.n_rec, 0, None, sc.kept.data_ptr(),
                                      sc.n_kept.data_ptr(), sc.ws.data_ptr(), sc.ws.numel(),
                                      self.compute.cuda_stream)
            _lib.check(rc, "pareto")
            sc.n_host.copy_(sc.n_kept, non_blocking=True)
            slot["count"].record(self.compute)
        ticket = self._ticket
        self._ticket += 1
        self._pending.append((s, ticket))
        return ticket

    def _finish_oldest(self) -> None:
        s, ticket = self._pending.popleft()
        slot = self.slots[s]
        slot["count"].synchronize()
        sc = slot["scratch"]
        n = int(sc.n_host[0])
        with torch.cuda.stream(self.tail):
            self.tail.wait_event(slot["count"])
            rows = front_rows(sc.kept[:n], slot["out"])
            host = torch.empty(rows.shape, dtype=rows.dtype, pin_memory=True) \
                if slot.get("host") is None or slot["host"].numel() < rows.numel() \
                else slot["host"]
            slot["host"] = host
            dst = host.view(-1)[: rows.numel()].view(rows.shape)
            dst.copy_(rows, non_blocking=True)
            slot["tail"].record(self.tail)
        slot["tail"].synchronize()
        self._done[ticket] = dst.numpy().copy()

    def result(self, ticket: int) -> np.ndarray:
        """Front rows of a submitted sweep (waits for it)."""
        while ticket not in self._done:
            if not self._pending:
                raise KeyError(f"unknown ticket {ticket}")
            self._finish_oldest()
        return self._done.pop(ticket)

    def drain(self) -> None:
        while self._pending:
            self._finish_oldest()


_ = ctypes
