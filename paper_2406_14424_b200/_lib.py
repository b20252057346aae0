"""ctypes binding of the C ABI in include/gearserve_b200.h.

This is the only place the package touches the native library.  There is no
CPU fallback: if the shared library is missing or no CUDA device is visible,
every compute call raises instead of silently running elsewhere.  PyTorch is
used for device memory (caching allocator), pinned host buffers and the
current CUDA stream; no torch type crosses the C boundary.
"""

from __future__ import annotations

import ctypes
import threading
from ctypes import POINTER, c_double, c_int32, c_int64, c_size_t, c_uint8, c_uint32, c_void_p
from pathlib import Path

import numpy as np
import torch

import os

# GS_LIB_PATH selects another build of the same C ABI (e.g. the phase-timing
# build tools/phase_probe.py makes); the default is the in-tree release build.
LIB_PATH = Path(os.environ.get("GS_LIB_PATH") or
                Path(__file__).resolve().with_name("libgearserve_b200.so"))

GS_OK = 0
GS_EINVAL = -1
GS_ECUDA = -2
GS_EWORKSPACE = -3
GS_EUNSUPPORTED = -4

GS_CERT_MARGIN = 0
GS_CERT_MAX_SOFTMAX = 1
GS_CERT_ENTROPY = 2
CERT_KINDS = {"margin": GS_CERT_MARGIN, "max_softmax": GS_CERT_MAX_SOFTMAX,
              "entropy": GS_CERT_ENTROPY}

GS_F32 = 0
GS_F64 = 1
GS_BF16 = 2
DTYPES = {torch.float32: GS_F32, torch.float64: GS_F64, torch.bfloat16: GS_BF16}


class gs_grid_info(ctypes.Structure):
    _fields_ = [("n_configs", c_int64), ("n_cells", c_int64), ("side_cells", c_int64),
                ("n_structures", c_int32), ("max_len", c_int32), ("workspace_bytes", c_size_t),
                ("build_launches", c_int32), ("eval_launches", c_int32), ("fast_path", c_int32),
                ("reserved", c_int32)]


GS_JSONL_MAX_MODELS = 64


class gs_jsonl_info(ctypes.Structure):
    _fields_ = [("n_records", c_int64), ("n_models", c_int32),
                ("width", c_int32 * GS_JSONL_MAX_MODELS),
                ("model_ids", (ctypes.c_char * 64) * GS_JSONL_MAX_MODELS),
                ("err_line", c_int64), ("error", ctypes.c_char * 256)]


# symbol -> argtypes (all return c_int unless listed in _RESTYPES)
_SIGNATURES = {
    "gs_version": [],
    "gs_flush_l2": [c_void_p, c_size_t, c_int32, c_void_p],
    "gs_strerror": [c_int32],
    "gs_last_cuda_error": [],
    "gs_eval_encoded_workspace": [c_int64, c_int32, c_int64, c_int32, POINTER(c_size_t)],
    "gs_eval_encoded": [c_void_p, c_void_p, c_int64, c_int32, c_void_p, c_void_p, c_void_p,
                        c_int64, c_int32, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                        c_size_t, c_void_p],
    "gs_grid_plan": [c_int64, c_int32, POINTER(c_int32), POINTER(gs_grid_info)],
    "gs_grid_build": [c_void_p, c_void_p, c_int64, c_int32, c_void_p, POINTER(c_int32),
                      c_void_p, c_size_t, c_int32, c_void_p],
    "gs_grid_accumulate": [c_void_p, c_void_p, c_int64, c_int64, c_int32, c_void_p,
                           POINTER(c_int32), c_void_p, c_size_t, c_int32, c_void_p],
    "gs_grid_finish": [c_int64, c_int32, POINTER(c_int32), c_void_p, c_size_t, c_void_p],
    "gs_quantiles_workspace": [c_int64, c_int32, POINTER(c_size_t)],
    "gs_quantiles": [c_void_p, c_int64, c_int64, c_void_p, c_int32, c_void_p, c_void_p, c_size_t,
                     c_void_p],
    "gs_jsonl_open": [ctypes.c_char_p, c_int32, POINTER(c_void_p), POINTER(gs_jsonl_info)],
    "gs_jsonl_read": [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p],
    "gs_jsonl_close": [c_void_p],
    "gs_grid_sweep_batched": [c_void_p, c_void_p, c_int64, c_int64, c_int32, c_void_p,
                              POINTER(c_int32), c_void_p, c_void_p, c_void_p, c_void_p, c_void_p],
    "gs_grid_eval": [c_int64, c_int32, POINTER(c_int32), c_void_p, c_int64, c_int64, c_void_p,
                     c_void_p, c_void_p, c_void_p, c_void_p, c_size_t, c_void_p],
    "gs_grid_decode": [c_int32, POINTER(c_int32), c_void_p, c_void_p, c_int64, c_void_p,
                       c_void_p, c_void_p, c_void_p],
    "gs_pareto_counts_workspace": [c_int64, c_int64, POINTER(c_size_t)],
    "gs_pareto_counts": [c_void_p, c_void_p, c_int64, c_int64, c_int64, c_void_p, c_void_p,
                         c_void_p, c_void_p, c_size_t, c_void_p],
    "gs_pareto_generic": [c_void_p, c_void_p, c_int64, c_void_p, c_void_p],
    "gs_certainty": [c_void_p, c_int32, c_int64, c_int32, c_int64, c_void_p, c_int32, c_void_p,
                     c_void_p],
    "gs_stage_step_workspace": [c_int64, POINTER(c_size_t)],
    "gs_stage_step": [c_void_p, c_int32, c_int64, c_int32, c_int64, c_int32, c_void_p, c_void_p,
                      c_void_p, c_void_p, c_void_p, c_void_p, c_double, c_void_p, c_void_p,
                      c_void_p, c_int64, c_void_p, c_void_p, c_size_t, c_void_p],
    "gs_stage_gate": [c_void_p, c_void_p, c_int64, c_int32, c_void_p, c_void_p, c_void_p,
                      c_void_p, c_int64, c_void_p, c_void_p, c_void_p, c_void_p, c_double,
                      c_void_p, c_void_p, c_void_p, c_size_t, c_void_p],
    "gs_engine_run": [c_void_p, c_int32, c_void_p],
    "gs_front5_plan": [c_int64, POINTER(c_int32), c_void_p],
    "gs_front5_prepare": [c_void_p, c_void_p, c_int64, c_void_p, POINTER(c_int32), c_void_p,
                          c_size_t, c_void_p],
    "gs_front5_pass1": [c_int64, POINTER(c_int32), c_void_p, c_int32, c_int32, c_void_p, c_size_t,
                        c_void_p],
    "gs_front5_select": [c_int64, POINTER(c_int32), c_void_p, c_size_t, c_void_p, c_void_p],
    "gs_front5_pass2": [c_int64, POINTER(c_int32), c_void_p, c_int32, c_int32, c_void_p, c_size_t,
                        c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_void_p],
    "gs_sample_cascades": [c_int32, c_void_p, c_void_p, c_void_p, c_void_p, c_int32, c_void_p],
    "gs_stage_gate_packed_bytes": [c_int64, POINTER(c_size_t), POINTER(c_size_t),
                                   POINTER(c_size_t)],
    "gs_stage_gate_packed": [c_void_p, c_void_p, c_int64, c_int32, c_void_p, c_int64, c_double,
                             c_void_p, c_void_p, c_size_t, c_int32, c_void_p],
    "gs_head_certainty": [c_void_p, c_void_p, c_void_p, c_int64, c_int32, c_int32, c_int32, c_void_p,
                          c_void_p, c_void_p],
}
_RESTYPES = {"gs_strerror": ctypes.c_char_p, "gs_last_cuda_error": ctypes.c_char_p,
             "gs_jsonl_close": None}

_lock = threading.Lock()
_lib: ctypes.CDLL | None = None


def load() -> ctypes.CDLL:
    """Load libgearserve_b200.so (built in-tree by __graft_entry__.build())."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise RuntimeError(
                    f"{LIB_PATH.name} is not built; run `python -c 'import __graft_entry__ as g; "
                    f"g.build()'` (there is no CPU fallback)")
            lib = ctypes.CDLL(str(LIB_PATH))
            for name, argtypes in _SIGNATURES.items():
                fn = getattr(lib, name)
                fn.argtypes = argtypes
                fn.restype = _RESTYPES.get(name, ctypes.c_int)
            _lib = lib
    return _lib


def exported_symbols() -> list[str]:
    return list(_SIGNATURES)


def device() -> torch.device:
    """The CUDA device every kernel runs on; raises when there is none."""
    if not torch.cuda.is_available():
        raise RuntimeError("gearserve-b200 kernels need a CUDA device (sm_100a); "
                           "there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def stream_ptr() -> int:
    """The current CUDA stream of the current device as an integer handle."""
    if _raw_stream is not None:
        return _raw_stream(torch.cuda.current_device())
    return torch.cuda.current_stream().cuda_stream


def check(rc: int, what: str) -> None:
    if rc == GS_OK:
        return
    lib = load()
    msg = lib.gs_strerror(rc).decode()
    if rc == GS_ECUDA:
        raise RuntimeError(f"{what}: {msg}: {lib.gs_last_cuda_error().decode()}")
    if rc in (GS_EINVAL, GS_EWORKSPACE):
        raise ValueError(f"{what}: {msg}")
    raise ValueError(f"{what}: {msg} (shape outside the kernel's supported range)")


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def workspace(nbytes: int) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device())


def int32_array(values) -> ctypes.Array:
    vals = [int(v) for v in values]
    return (c_int32 * len(vals))(*vals)


def to_device(a, dtype: torch.dtype) -> torch.Tensor:
    """numpy / tensor -> contiguous device tensor of dtype (H2D through pinned
    memory when the source is on the host)."""
    dev = device()
    if isinstance(a, torch.Tensor):
        t = a
        if t.device.type != "cuda":
            t = t.to(dtype).contiguous().pin_memory().to(dev, non_blocking=True)
        return t.to(dev, dtype).contiguous()
    arr = np.ascontiguousarray(a)
    t = torch.from_numpy(arr).to(dtype)
    if t.numel() > 0:
        t = t.pin_memory()
    return t.to(dev, non_blocking=True)


def to_numpy(t: torch.Tensor) -> np.ndarray:
    return t.cpu().numpy()


__all__ = [name for name in globals() if not name.startswith("_")]
_ = (c_uint8, c_uint32)


def row_stride(t: torch.Tensor) -> int:
    """Row pitch (elements) of a 2-D row-major matrix; size-1 leading dims
    may carry any stride (numpy broadcasting views), so use the width."""
    return int(t.stride(0)) if t.shape[0] > 1 else int(t.shape[1])
