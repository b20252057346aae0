"""Build this package's plan / trace / validation objects for the replay
scenarios of golden_inputs.replay_cases() (the golden generator builds the
reference's own objects from the same data)."""

import numpy as np

import golden_inputs as gi


def build(case):
    from paper_2406_14424_b200 import replay, synth
    from paper_2406_14424_b200.types import (Cascade, Gear, GearPlan, Placement, Replica,
                                             ValidationArrays, WorkloadTrace)
    prof = synth.make_profiles(n_models=case["profiles"]["n_models"],
                               cost_ratios=tuple(case["profiles"]["cost_ratios"]))
    n, easy, vseed = case["val"]
    cert, corr = synth.validation_matrices(len(prof), n, easy, vseed)
    val = ValidationArrays(prof.model_ids, certainty=cert, correct=corr)
    kind, args = next(iter(case["trace"].items()))
    if kind == "bursty":
        seconds, seed, max_qps = args
        trace = replay.scale_trace(synth.trace_from_counts(gi.bursty_counts(seconds, seed)),
                                   max_qps)
    elif kind == "constant":
        trace = synth.constant_rate_trace(*args)
    elif kind == "zeros":
        trace = WorkloadTrace(np.zeros(args[0], dtype=np.int64), duration_us=args[1])
    else:
        trace = synth.step_trace([tuple(x) for x in args])
    sp = case["plan"]
    gears = tuple(Gear(cascade=Cascade(stages=tuple(g["stages"]), thresholds=tuple(g["thresholds"])),
                       min_queue_length=dict(g["min_q"]),
                       load_weights={m: dict(w) for m, w in g["weights"].items()})
                  for g in sp["gears"])
    plan = GearPlan(placement=Placement([Replica(*r) for r in sp["replicas"]]), slo=None,
                    qps_max=sp["qps_max"], gears=gears)
    cfg = replay.EngineConfig(seed=case["seed"], measure_period_us=case["period"],
                              alpha=case["alpha"], initial_gear_index=case["initial_gear"],
                              enable_ticks=case["ticks"])
    return prof, val, trace, plan, cfg
