"""Timing of the fused tensor-core head + certainty (gs_head_certainty) vs
the unfused torch path (cuBLAS bf16 GEMM -> logits -> gs_certainty), CUDA
events, L2 not flushed (features 268 MB > L2 at the large shape)."""
import math, sys
import torch
sys.path.insert(0, ".")
from paper_2406_14424_b200.head import head_certainty
from paper_2406_14424_b200.cascades import certainty_rows

for B, N, K in ((65536, 1000, 2048), (65536, 1000, 512), (262144, 1000, 512)):
    f = torch.randn(B, K, device="cuda").to(torch.bfloat16)
    w = (torch.randn(N, K, device="cuda") / math.sqrt(K)).to(torch.bfloat16)
    def fused():
        return head_certainty(f, w, kind="entropy")
    def unfused():
        return certainty_rows(f @ w.T, kind="entropy")
    for name, fn in (("fused", fused), ("unfused", unfused)):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10):
            fn()
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 10
        print(f"B={B} N={N} K={K} {name:8s} {ms*1e3:9.1f} us  {2*B*N*K/ms/1e9:8.1f} TFLOP/s  {B/ms/1e3:8.1f} Mrows/s",
              flush=True)
