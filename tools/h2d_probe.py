"""H2D of the config-2 certainty matrix [1M, 4] f64 from pinned host memory:
the whole matrix (32 MB) vs only the three columns the grid path reads
(cudaMemcpy2DAsync, 24 of every 32 bytes), and the whole matrix as two
halves on two streams at once (both copy engines), CUDA events."""
import torch
from cuda.bindings import runtime as rt

N = 1_000_000
h = torch.rand(N, 4, dtype=torch.float64).pin_memory()
d = torch.empty(N, 4, dtype=torch.float64, device="cuda")
s = torch.cuda.current_stream()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def full():
    d.copy_(h, non_blocking=True)


def cols3():
    err, = rt.cudaMemcpy2DAsync(d.data_ptr(), 32, h.data_ptr(), 32, 24, N,
                                rt.cudaMemcpyKind.cudaMemcpyHostToDevice, s.cuda_stream)
    assert err == rt.cudaError_t.cudaSuccess, err


s2 = torch.cuda.Stream()


def halves():
    e = torch.cuda.Event()
    e.record(s)
    s2.wait_event(e)
    d[: N // 2].copy_(h[: N // 2], non_blocking=True)
    with torch.cuda.stream(s2):
        d[N // 2:].copy_(h[N // 2:], non_blocking=True)
    e2 = torch.cuda.Event()
    e2.record(s2)
    s.wait_event(e2)


for name, fn, nbytes in (("full 32 MB", full, 32e6), ("3 of 4 columns (2D)", cols3, 24e6),
                         ("two halves, two streams", halves, 32e6)):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a.record()
    for _ in range(10):
        fn()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 10
    print(f"{name:24s} {ms * 1e3:8.1f} us  {nbytes / (ms * 1e-3) / 1e9:6.1f} GB/s moved", flush=True)
torch.cuda.synchronize()
assert torch.equal(d[:, :3].cpu(), h[:, :3])
