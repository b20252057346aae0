"""Config 5's device replay (8 replica groups of the bursty trace), launched
twice (for ncu: -k regex:engine_kernel -s 1 -c 1)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2406_14424_b200 import replay, synth
from paper_2406_14424_b200.types import ValidationArrays

groups = 8
trace = replay.scale_trace(synth.trace_from_counts(synth.bursty_counts(1200, 0)), 7600.0)
parts = replay.split_round_robin(trace, groups)
prof, plan = synth.replica_group_plan(qps_max=7600.0 / groups)
cert, corr = synth.validation_matrices(4, 100_000, 0.8, 5)
dp = replay.DevicePlan(plan, prof, ValidationArrays(prof.model_ids, certainty=cert, correct=corr))
jobs = [replay.Job(dp, p.arrivals, p.duration_us, replay.EngineConfig(seed=g)) for g, p in enumerate(parts)]
prep = replay.Prepared(jobs)
for _ in range(2):
    prep.run()
torch.cuda.synchronize()
print("done", sum(r.completed for r in prep.results()))
