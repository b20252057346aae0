"""The hot-path entry points as torch operators (torch.ops.gearserve_b200.*).

libgearserve_b200_torch.so (csrc/gs_torch_ops.cpp, built in-tree by
_build.build_torch_ops) registers them with TORCH_LIBRARY over the C ABI, so
the kernels are visible to torch's dispatcher: CUDA tensors in, tensors from
the caching allocator out, launched on the current stream.  There is no CPU
kernel: a CPU tensor raises (no fallback).

    ops = torch_ops.load()
    acc, cost, frac = ops.evaluate_encoded(cert, corr, stage_model, thr, n_stages, cost1)
    acc, cost, frac, n_correct = ops.grid_sweep(cert, corr, grids_flat, grid_len, cost1)
    front = ops.pareto_counts(n_correct, cost, n_rec)
    cert = ops.certainty(logits, 2)       # GS_CERT_* kind
    q = ops.quantiles(column, [0.1, 0.5])
    cert = ops.head_certainty(features_bf16, weight_bf16, bias_f32, 2)
"""

from __future__ import annotations

from pathlib import Path

import torch

from . import _lib

LIB = Path(__file__).resolve().parent / "libgearserve_b200_torch.so"
OPS = ("evaluate_encoded", "grid_sweep", "pareto_counts", "certainty", "quantiles", "head_certainty")
_loaded = False


def load():
    """Load the operator library (once) and return torch.ops.gearserve_b200."""
    global _loaded
    if not _loaded:
        if not LIB.exists():
            raise RuntimeError(f"{LIB.name} is not built (paper_2406_14424_b200._build.build_torch_ops)")
        _lib.load()  # the kernel library it links, loaded from the same directory
        torch.ops.load_library(str(LIB))
        _loaded = True
    return torch.ops.gearserve_b200
