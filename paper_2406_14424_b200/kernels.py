"""Drop-in for gearserve.kernels (/root/reference/pkg/src/gearserve/kernels.py).

evaluate_encoded keeps the reference signature and return contract
(src/kernels.py:93-108): positional arrays coerced to f64 / u8 / i32 / f64 /
i32 / f64, freshly allocated numpy outputs
(accuracy[n_casc], mean_cost[n_casc], forward_frac[n_casc, max_len]).
It runs the sm_100a list-path kernel (csrc/gs_eval.cu) and is bit-identical
to the reference's numba walk (src/kernels.py:39-62).

The reference picks numba or numpy through GEARSERVE_DISABLE_NUMBA
(:35-36).  This build has exactly one backend, the CUDA kernel: HAS_NUMBA is
False and numba_enabled() always answers False, so callers probing the flag
keep working, and there is no CPU path to fall back to.

evaluate_encoded_device is the device-resident variant: torch CUDA tensors
in, torch CUDA tensors out, no host round trip.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib

HAS_NUMBA = False


def numba_enabled() -> bool:
    """Always False: the B200 build has a single (CUDA) backend."""
    return False


def _validate_encoded(n_models: int, stage_model: np.ndarray, n_stages: np.ndarray,
                      thresholds: np.ndarray) -> None:
    if stage_model.ndim != 2 or thresholds.shape != stage_model.shape:
        raise ValueError("stage_model and thresholds must both be [n_casc, max_len]")
    if n_stages.shape != (stage_model.shape[0],):
        raise ValueError("n_stages must be [n_casc]")
    if stage_model.size == 0:
        return
    max_len = stage_model.shape[1]
    if np.any(n_stages > max_len) or np.any(n_stages < 0):
        raise IndexError("n_stages exceeds the encoded cascade width")
    used = np.arange(max_len)[None, :] < n_stages[:, None]
    sm = stage_model[used]
    if sm.size and (sm.min() < -n_models or sm.max() >= n_models):
        raise IndexError(f"stage model index out of range for {n_models} models")
    if sm.size and sm.min() < 0:
        # numpy would wrap negative indices; the encoding pads with -1 only
        # past n_stages, so a negative live entry is malformed input
        raise IndexError("negative stage model index inside n_stages")


def evaluate_encoded_device(certainty: torch.Tensor, correct: torch.Tensor,
                            stage_model: torch.Tensor, thresholds: torch.Tensor,
                            n_stages: torch.Tensor, cost1: torch.Tensor):
    """Device-resident evaluate_encoded: CUDA tensors in (f64, u8, i32, f64,
    i32, f64), CUDA tensors out; runs on the current stream."""
    lib = _lib.load()
    dev = _lib.device()
    n_rec, n_models = int(certainty.shape[0]), int(certainty.shape[1])
    n_casc, max_len = int(stage_model.shape[0]), int(stage_model.shape[1])
    acc = torch.zeros(n_casc, dtype=torch.float64, device=dev)
    cost = torch.zeros(n_casc, dtype=torch.float64, device=dev)
    frac = torch.zeros((n_casc, max_len), dtype=torch.float64, device=dev)
    if n_casc == 0:
        return acc, cost, frac
    if n_rec == 0:
        raise ZeroDivisionError("division by zero")
    nbytes = ctypes.c_size_t()
    _lib.check(lib.gs_eval_encoded_workspace(n_rec, n_models, n_casc, max_len,
                                             ctypes.byref(nbytes)), "evaluate_encoded")
    ws = _lib.workspace(nbytes.value)
    rc = lib.gs_eval_encoded(
        certainty.data_ptr(), correct.data_ptr(), n_rec, n_models, stage_model.data_ptr(),
        thresholds.data_ptr(), n_stages.data_ptr(), n_casc, max_len, cost1.data_ptr(),
        acc.data_ptr(), cost.data_ptr(), frac.data_ptr(), ws.data_ptr(), ws.numel(),
        _lib.stream_ptr())
    _lib.check(rc, "evaluate_encoded")
    return acc, cost, frac


def evaluate_encoded(certainty: np.ndarray, correct: np.ndarray,
                     stage_model: np.ndarray, thresholds: np.ndarray,
                     n_stages: np.ndarray, cost1: np.ndarray):
    """Score encoded cascades on the GPU.

    Returns (accuracy[n_casc], mean_cost[n_casc], forward_frac[n_casc, max_len])
    as numpy f64 arrays, bit-identical to the reference.
    """
    certainty = np.ascontiguousarray(certainty, dtype=np.float64)
    correct = np.ascontiguousarray(correct, dtype=np.uint8)
    stage_model = np.ascontiguousarray(stage_model, dtype=np.int32)
    thresholds = np.ascontiguousarray(thresholds, dtype=np.float64)
    n_stages = np.ascontiguousarray(n_stages, dtype=np.int32)
    cost1 = np.ascontiguousarray(cost1, dtype=np.float64)
    n_models = certainty.shape[1] if certainty.ndim == 2 else 0
    _validate_encoded(n_models, stage_model, n_stages, thresholds)
    n_casc = stage_model.shape[0]
    if n_casc == 0:
        return (np.zeros(0), np.zeros(0), np.zeros((0, stage_model.shape[1])))
    if certainty.shape[0] == 0:
        raise ZeroDivisionError("division by zero")
    outs = evaluate_encoded_device(
        _lib.to_device(certainty, torch.float64), _lib.to_device(correct, torch.uint8),
        _lib.to_device(stage_model, torch.int32), _lib.to_device(thresholds, torch.float64),
        _lib.to_device(n_stages, torch.int32), _lib.to_device(cost1, torch.float64))
    return tuple(_lib.to_numpy(t) for t in outs)
