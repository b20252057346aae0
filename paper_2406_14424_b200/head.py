"""A cascade stage's classifier head on the tensor cores, fused with the
stage step's certainty (csrc/gs_head.cu, gs_head_certainty).

north_star: "Tensor cores are used only for the dense classifier GEMMs
inside each cascade model".  The reference's stage runs a model and takes
cascades.certainty of its scores (src/serving.py:79-97, src/cascades.py:20-28);
here the head's GEMM (bf16 features x bf16 weight, f32 accumulation in TMEM)
and the certainty run as one kernel, so a stage step reads the features and
the weight and writes one f64 per row.  The gate and the compaction of the
deferred rows then run on the certainties (stage.stage_gate)."""

from __future__ import annotations

import torch

from . import _lib


def head_certainty(features: torch.Tensor, weight: torch.Tensor, bias: torch.Tensor | None = None,
                   kind: str = "entropy", logits: bool = False):
    """certainty[B] (CUDA f64) of softmax(features @ weight.T + bias) rows
    (or of the logits for kind="margin"); with logits=True also returns the
    f32 logits [B, N].  features [B, K] and weight [N, K] are bf16 CUDA
    tensors (converted if not), K a multiple of 64."""
    if kind not in _lib.CERT_KINDS:
        raise ValueError(f"unknown certainty kind {kind!r}")
    dev = _lib.device()
    f = _lib.to_device(features, torch.bfloat16)
    w = _lib.to_device(weight, torch.bfloat16)
    if f.ndim != 2 or w.ndim != 2 or f.shape[1] != w.shape[1]:
        raise ValueError("features [B, K] and weight [N, K] must share K")
    if f.shape[1] % 64 != 0:
        raise ValueError("the feature width must be a multiple of 64")
    b = None if bias is None else _lib.to_device(bias, torch.float32)
    if b is not None and b.numel() != w.shape[0]:
        raise ValueError("bias must hold one value per class")
    n, n_cls = int(f.shape[0]), int(w.shape[0])
    cert = torch.empty(n, dtype=torch.float64, device=dev)
    out = torch.empty((n, n_cls), dtype=torch.float32, device=dev) if logits else None
    rc = _lib.load().gs_head_certainty(f.data_ptr(), w.data_ptr(), None if b is None else b.data_ptr(), n,
                                       n_cls, int(f.shape[1]), _lib.CERT_KINDS[kind], cert.data_ptr(),
                                       None if out is None else out.data_ptr(), _lib.stream_ptr())
    _lib.check(rc, "head_certainty")
    return (cert, out) if logits else cert


def head_stage_step(features: torch.Tensor, weight: torch.Tensor, thr, bias: torch.Tensor | None = None,
                    is_last=None, *, kind: str = "entropy", forward_features: bool = True,
                    near_eps: float = 1e-5):
    """One online cascade stage on the tensor cores: the head's certainty per
    row (head_certainty), then the stage gate on it — stop when
    cert >= thr (or the stage is the last), deferred rows compacted in batch
    order and, with forward_features, their feature rows gathered into the
    next stage's contiguous batch (stage.stage_step on the [n, 1] certainty
    column: a one-class row's margin is its value).  near_eps lists the rows
    whose certainty lies within it of the threshold (the head's f32
    accumulation and ex2 put its certainty within ~5e-6 of a float64
    recomputation, so the default band is wider than the score path's)."""
    from .stage import stage_step
    f = _lib.to_device(features, torch.bfloat16)
    cert = head_certainty(f, weight, bias, kind=kind)
    res = stage_step(cert.view(-1, 1), thr, is_last, kind="margin", payload=f if forward_features else None,
                     near_eps=near_eps)
    return res
