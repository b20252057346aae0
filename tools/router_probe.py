"""Where a batch-4 StageRouter.finish_batch call spends its time: the whole
call, the gate's C call alone, and pieces of the host side (host wall clock)."""
import sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2406_14424_b200 import _lib, synth
from paper_2406_14424_b200.engine import GearTables, Item, StageRouter

prof, plan = synth.replica_group_plan(qps_max=950.0)
cert, corr = synth.validation_matrices(4, 100_000, 0.8, 5)
reps = list(plan.placement.replicas)
ids = list(prof.model_ids)
devs = []
for r in reps:
    if r.device_id not in devs:
        devs.append(r.device_id)
tables = GearTables.from_gears(plan.gears, [(r.replica_id, r.model_id) for r in reps], {m: j for j, m in enumerate(ids)})
router = StageRouter(tables, cert, corr, [devs.index(r.device_id) for r in reps], seed=0)
rng = np.random.default_rng(0)
N = 5000
batches = [[Item(c * 4 + k, int(rng.integers(0, 100_000)), 0, int(rng.integers(0, len(plan.gears))), 0) for k in range(4)] for c in range(N)]


def timeit(name, fn, n=N):
    for i in range(50):
        fn(i)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for i in range(n):
        fn(i)
    dt = (time.perf_counter() - t) / n * 1e6
    print(f"{name:40s} {dt:8.2f} us per call", flush=True)


timeit("finish_batch (batch 4)", lambda i: router.finish_batch(0, batches[i], 10))
rows = np.array([3, 7, 11, 19], np.int64); model = np.zeros(4, np.int32); thr = np.full(4, 0.5); last = np.zeros(4, bool)
timeit("GateBatcher.gate (batch 4)", lambda i: router.gate.gate(rows, model, thr, last))
timeit("_lib.stream_ptr()", lambda i: _lib.stream_ptr())
timeit("torch.cuda.current_stream()", lambda i: torch.cuda.current_stream())
lib = _lib.load()
g = router.gate
args = (g.cert.data_ptr(), g.corr.data_ptr(), g.n_rec, g.n_models, g.h_in.data_ptr(), 4, g.near_eps,
        g.h_out.data_ptr(), g.d_buf.data_ptr(), g.d_buf.numel(), 1, _lib.stream_ptr())
timeit("gs_stage_gate_packed, cached args", lambda i: lib.gs_stage_gate_packed(*args))
timeit("cudaDeviceSynchronize (torch)", lambda i: torch.cuda.synchronize())
