"""Config 4a: the exact Pareto front of a five-model cascade over
1000-level threshold grids (csrc/gs_front5.cu).

The configs are every threshold tuple (k0, k1, k2, k3) of the full cascade
m0 -> m1 -> m2 -> m3 -> m4 over the per-model grids (g0 g1 g2 g3 of them,
~1e12 at 1000 levels), each scored as the reference's walk scores it
(/root/reference/pkg/src/gearserve/kernels.py:39-62); the output is the
reference's pareto_filter front over (accuracy, mean_cost), exact ties kept
(src/cascades.py:116-129), in config order, with accuracy, mean_cost and
forward_frac as evaluate_encoded returns them.  Config index =
((k0 g1 + k1) g2 + k2) g3 + k3 -- the offset of the config inside the full
cascade's block of gridsweep's enumeration.

Sharding: configs split by k0 (pass1 / pass2 take a k0 range); the
per-accuracy minimum costs are reduced with MIN across ranks between the
passes (mincost()), and the ranks' fronts are disjoint slices of the answer.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib


class gs_front5_info(ctypes.Structure):
    _fields_ = [("n_configs", ctypes.c_int64), ("workspace_bytes", ctypes.c_size_t),
                ("mincost_offset", ctypes.c_size_t), ("front_offset", ctypes.c_size_t),
                ("ties_offset", ctypes.c_size_t), ("min_index_offset", ctypes.c_size_t),
                ("k0_count", ctypes.c_int32), ("bucket_shift", ctypes.c_int32)]


@dataclass
class Front:
    index: np.ndarray          # u64 config index (ascending)
    accuracy: np.ndarray       # f64
    mean_cost: np.ndarray      # f64
    forward_frac: np.ndarray   # f64 [n, 5]
    n_correct: np.ndarray      # u32
    n_configs: int


def k0_cuts(cert0, grid0, world: int) -> np.ndarray:
    """Cut points [world + 1] of k0 = 0..g0 for sharding the passes over the
    ranks with about equal work each.  A k0's rows stream the records with
    b0 <= k0, so its cost grows with R(k0) = #(b0 <= k0); measured on one
    B200 (config 4a) a k0 near R = 0.6 n costs about twice one near R = 0,
    modelled as 1 + 2 R(k0) / n.  Equal-count cuts would leave the last rank
    about 1.4x the mean at 8 ranks."""
    g = np.asarray(grid0, dtype=np.float64)
    x = np.asarray(cert0, dtype=np.float64)
    n = max(1, x.size)
    g0 = int(g.size)
    b0 = np.searchsorted(g, x, side="right")  # #(g <= x), the kernel's bin
    r = np.cumsum(np.bincount(b0, minlength=g0 + 1))[:g0]  # R(k0) for k0 = 0..g0-1
    w = 1.0 + 2.0 * r / n
    cw = np.concatenate([[0.0], np.cumsum(w)])
    cuts = np.searchsorted(cw, cw[-1] * np.arange(world + 1) / world, side="left")
    cuts[0], cuts[-1] = 0, g0
    return np.maximum.accumulate(np.clip(cuts, 0, g0)).astype(np.int64)


class Front5:
    """Prepared records (bins, sorted keys, side tables) of one validation
    set and its grids; pass1 / select / pass2 compute the front."""

    def __init__(self, certainty, correct, grids, cost1):
        self.cert = _lib.to_device(certainty, torch.float64)
        self.corr = _lib.to_device(correct, torch.uint8)
        if self.cert.ndim != 2 or self.cert.shape[1] != 5 or \
                tuple(self.corr.shape) != tuple(self.cert.shape):
            raise ValueError("certainty and correct must both be [n_records, 5]")
        if len(grids) != 5:
            raise ValueError("need 5 grids")
        host = []
        for j, g in enumerate(grids):
            g = np.asarray(g.cpu() if isinstance(g, torch.Tensor) else g, dtype=np.float64)
            if g.ndim != 1 or g.size == 0 or np.any(np.diff(g) <= 0):
                raise ValueError(f"grid {j} must be a non-empty strictly increasing 1-D array")
            host.append(g)
        self.n_rec = int(self.cert.shape[0])
        self.grids_host = host
        self._cert0 = self.cert[:, 0].cpu().numpy()  # k0_cuts' record bins
        self.grid_len = [int(g.size) for g in host]
        self._glen = _lib.int32_array(self.grid_len)
        self.grids = _lib.to_device(np.concatenate(host[:4]), torch.float64)
        self.cost1 = _lib.to_device(np.asarray(cost1, dtype=np.float64), torch.float64)
        if self.cost1.numel() != 5:
            raise ValueError("cost1 must have 5 entries")
        lib = _lib.load()
        info = gs_front5_info()
        _lib.check(lib.gs_front5_plan(self.n_rec, self._glen, ctypes.byref(info)), "front5 plan")
        self.info = info
        self.n_configs = int(info.n_configs)
        self.ws = torch.empty(int(info.workspace_bytes), dtype=torch.uint8, device=_lib.device())
        self.prepare()

    def k0_cuts(self, world: int) -> np.ndarray:
        """k0 ranges of about equal work for `world` ranks (k0_cuts)."""
        return k0_cuts(self._cert0, self.grids_host[0], world)

    def prepare(self) -> None:
        """Bin and sort the records, build the side tables, reset mincost."""
        _lib.check(_lib.load().gs_front5_prepare(
            self.cert.data_ptr(), self.corr.data_ptr(), self.n_rec, self.grids.data_ptr(),
            self._glen, self.ws.data_ptr(), self.ws.numel(), _lib.stream_ptr()), "front5 prepare")

    def _range(self, k0_begin, k0_end):
        k0_end = self.grid_len[0] if k0_end is None else int(k0_end)
        if not 0 <= int(k0_begin) <= k0_end <= self.grid_len[0]:
            raise ValueError("k0 range outside [0, g0]")
        return int(k0_begin), k0_end

    def pass1(self, k0_begin: int = 0, k0_end: int | None = None) -> None:
        b, e = self._range(k0_begin, k0_end)
        _lib.check(_lib.load().gs_front5_pass1(self.n_rec, self._glen, self.cost1.data_ptr(), b, e,
                                               self.ws.data_ptr(), self.ws.numel(),
                                               _lib.stream_ptr()), "front5 pass 1")

    def mincost(self) -> torch.Tensor:
        """The per-accuracy minimum cost keys (int64 [n_rec + 1], a view into
        the workspace): all-reduce them with MIN across ranks before select()."""
        off = int(self.info.mincost_offset)
        return self.ws[off: off + 8 * (self.n_rec + 1)].view(torch.int64)

    def select(self) -> int:
        """Fix the front's accuracies from mincost; returns how many there are."""
        n = torch.zeros(1, dtype=torch.int64, device=self.ws.device)
        _lib.check(_lib.load().gs_front5_select(self.n_rec, self._glen, self.ws.data_ptr(),
                                                self.ws.numel(), n.data_ptr(), _lib.stream_ptr()),
                   "front5 select")
        return int(n.item())

    def pass2(self, k0_begin: int = 0, k0_end: int | None = None, cap: int = 1 << 20):
        """Front configs with k0 in the range: (index u64, cost f64, counts
        u32 [n, 6] = correct, then reach before stages 0..4).  cap = 0: no
        list (the per-point summary, points(), only)."""
        b, e = self._range(k0_begin, k0_end)
        dev = self.ws.device
        if cap == 0:
            z = torch.zeros(1, dtype=torch.int64, device=dev)
            _lib.check(_lib.load().gs_front5_pass2(
                self.n_rec, self._glen, self.cost1.data_ptr(), b, e, self.ws.data_ptr(),
                self.ws.numel(), z.data_ptr(), z.data_ptr(), z.data_ptr(), z.data_ptr(), 0,
                _lib.stream_ptr()), "front5 pass 2")
            return None
        while True:
            idx = torch.empty(cap, dtype=torch.int64, device=dev)
            cost = torch.empty(cap, dtype=torch.float64, device=dev)
            cnt = torch.empty((cap, 6), dtype=torch.int32, device=dev)
            n = torch.zeros(1, dtype=torch.int64, device=dev)
            _lib.check(_lib.load().gs_front5_pass2(
                self.n_rec, self._glen, self.cost1.data_ptr(), b, e, self.ws.data_ptr(),
                self.ws.numel(), idx.data_ptr(), cost.data_ptr(), cnt.data_ptr(), n.data_ptr(), cap,
                _lib.stream_ptr()), "front5 pass 2")
            k = int(n.item())
            if k <= cap:
                return idx[:k], cost[:k], cnt[:k]
            cap = k  # rare: more tied front configs than room; redo with room

    def decode(self, index) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
        """Config indices -> evaluate_encoded's encoding (stage_model [n, 5]
        = 0..4, thresholds [n, 5], n_stages [n] = 5)."""
        idx = np.asarray(index, dtype=np.int64).reshape(-1)
        g = self.grid_len
        k = np.empty((idx.size, 4), dtype=np.int64)
        rest = idx.copy()
        for j in (3, 2, 1, 0):
            k[:, j] = rest % g[j]
            rest //= g[j]
        if np.any(rest != 0) or np.any(idx < 0):
            raise IndexError("config index outside the full cascade's block")
        thr = np.zeros((idx.size, 5))
        for j in range(4):
            thr[:, j] = self.grids_host[j][k[:, j]]
        sm = np.tile(np.arange(5, dtype=np.int32), (idx.size, 1))
        return sm, thr, np.full(idx.size, 5, dtype=np.int32)

    def _ws_view(self, off: int) -> torch.Tensor:
        return self.ws[off: off + 8 * (self.n_rec + 1)].view(torch.int64)

    def points(self):
        """After pass2: the front's distinct points in accuracy order --
        (n_correct, mean_cost, tied configs, smallest config index) as numpy
        arrays.  Every config of the front is one of these points."""
        key = self._ws_view(int(self.info.front_offset)).cpu().numpy()
        ties = self._ws_view(int(self.info.ties_offset)).cpu().numpy().view(np.uint64)
        mi = self._ws_view(int(self.info.min_index_offset)).cpu().numpy().view(np.uint64)
        on = np.flatnonzero(key != 0x7F7F7F7F7F7F7F7F)
        return on.astype(np.uint32), key[on].view(np.float64), ties[on], mi[on]

    def front(self, k0_begin: int = 0, k0_end: int | None = None) -> Front:
        """pass1 -> select -> pass2 on one device (k0_begin/k0_end: a sub-range
        of k0 whose front is wanted; the front of the sub-range's configs)."""
        self.prepare()
        self.pass1(k0_begin, k0_end)
        self.select()
        return assemble(*self.pass2(k0_begin, k0_end), self.n_rec, self.n_configs)


def assemble(idx: torch.Tensor, cost: torch.Tensor, counts: torch.Tensor, n_rec: int,
             n_configs: int) -> Front:
    """Host arrays in config order; accuracy and forward_frac from the
    integer counts with IEEE division (= the reference's count / n)."""
    order = torch.argsort(idx)
    i = idx[order].cpu().numpy().astype(np.uint64)
    c = cost[order].cpu().numpy()
    k = counts[order].cpu().numpy().astype(np.int64)
    n = float(n_rec)
    return Front(index=i, accuracy=k[:, 0] / n, mean_cost=c,
                 forward_frac=k[:, 1:6].astype(np.float64) / n,
                 n_correct=k[:, 0].astype(np.uint32), n_configs=n_configs)
