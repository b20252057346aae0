"""The tensor-core classifier head fused with the certainty (gs_head.cu) vs a
float64 torch reference of the same op (logits = features @ weight^T + bias,
then the certainty of each row)."""

import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _cert64(logits: torch.Tensor, kind: str) -> torch.Tensor:
    x = logits.double()
    if kind == "margin":
        if x.shape[1] == 1:
            return x[:, 0]
        t = torch.topk(x, 2, dim=1).values
        return t[:, 0] - t[:, 1]
    p = torch.softmax(x, dim=1)
    if kind == "max_softmax":
        return p.max(dim=1).values
    if x.shape[1] == 1:
        return torch.ones(x.shape[0], dtype=torch.float64, device=x.device)
    h = -(p * torch.log_softmax(x, dim=1)).sum(dim=1)
    return 1.0 - h / math.log(x.shape[1])


@pytest.mark.parametrize("B,N,K,bias", [(1000, 1000, 512, True), (300, 10, 64, False), (4097, 1000, 2048, True),
                                        (129, 257, 128, False), (64, 1, 64, True), (8192, 100, 256, False),
                                        (256, 5000, 64, True)])
@pytest.mark.parametrize("kind", ["entropy", "max_softmax", "margin"])
def test_head_certainty_vs_torch_f64(B, N, K, bias, kind):
    from paper_2406_14424_b200.head import head_certainty
    g = torch.Generator(device="cuda").manual_seed(B + N + K)
    f = (torch.randn(B, K, device="cuda", generator=g) * 0.5).to(torch.bfloat16)
    w = (torch.randn(N, K, device="cuda", generator=g) / math.sqrt(K) * 3).to(torch.bfloat16)
    b = torch.randn(N, device="cuda", generator=g) * 0.1 if bias else None
    cert, logits = head_certainty(f, w, b, kind=kind, logits=True)
    ref = f.double() @ w.double().T + (b.double() if bias else 0.0)
    # logits: f32 accumulation of bf16 products, any order
    assert torch.allclose(logits.double(), ref, rtol=1e-5, atol=1e-5)
    # certainty: the epilogue's math on its own logits, and end to end
    assert torch.allclose(cert, _cert64(logits, kind), rtol=0, atol=2e-6)
    assert torch.allclose(cert, _cert64(ref, kind), rtol=0, atol=2e-5)


def test_head_certainty_rejects_bad_shapes():
    from paper_2406_14424_b200.head import head_certainty
    f = torch.zeros(10, 100, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(ValueError):
        head_certainty(f, torch.zeros(5, 100, dtype=torch.bfloat16, device="cuda"))  # K % 64
    with pytest.raises(ValueError):
        head_certainty(torch.zeros(10, 64, dtype=torch.bfloat16, device="cuda"),
                       torch.zeros(5, 128, dtype=torch.bfloat16, device="cuda"))  # K mismatch


def test_head_stage_step_gates_and_forwards():
    """head -> gate -> compaction: the deferred rows are exactly the rows whose
    head certainty is below the threshold, in batch order, with their feature
    rows gathered; decisions differ from a float64 recomputation only inside
    the listed near-threshold band."""
    from paper_2406_14424_b200.head import head_certainty, head_stage_step
    g = torch.Generator(device="cuda").manual_seed(3)
    B, N, K = 5000, 1000, 512
    f = torch.randn(B, K, device="cuda", generator=g).to(torch.bfloat16)
    w = (torch.randn(N, K, device="cuda", generator=g) / math.sqrt(K) * 4).to(torch.bfloat16)
    cert = head_certainty(f, w, kind="entropy")
    thr = float(torch.quantile(cert, 0.35))
    res = head_stage_step(f, w, thr, kind="entropy")
    want = torch.nonzero(cert < thr).flatten()
    got = res.deferred_idx
    assert torch.equal(got, want)
    assert torch.equal(res.next_payload[: got.numel()], f[got])
    ref = _cert64(f.double() @ w.double().T, "entropy")
    differ = torch.nonzero((ref < thr) != (cert < thr)).flatten()
    near = set(res.near_idx.tolist())
    assert all(int(i) in near for i in differ)
