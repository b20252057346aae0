"""Golden vectors for the device replay engine, captured from the reference
engine.run (src/engine.py:452-520) on the scenarios of
golden_inputs.replay_cases().  Run where the reference imports:

    GEARSERVE_REF_SRC=/root/reference/pkg/src python tests/golden/make_golden_replay.py
"""

from __future__ import annotations

import json
import os
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF_SRC = os.environ.get("GEARSERVE_REF_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF_SRC)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from gearserve import engine as reng  # noqa: E402
from gearserve import formats as rformats  # noqa: E402
from gearserve import synth as rsynth  # noqa: E402
from gearserve import types as rt  # noqa: E402

sys.path.insert(0, str(HERE.parent))
import golden_inputs as gi  # noqa: E402


def ref_trace(spec):
    kind, args = next(iter(spec.items()))
    if kind == "bursty":
        seconds, seed, max_qps = args
        raw = rt.WorkloadTrace(gi.trace_from_counts(gi.bursty_counts(seconds, seed)))
        return rformats.scale_trace(raw, max_qps)
    if kind == "constant":
        return rsynth.constant_rate_trace(*args)
    if kind == "zeros":
        n, dur = args
        return rt.WorkloadTrace(np.zeros(n, dtype=np.int64), duration_us=dur)
    if kind == "step":
        return rsynth.step_trace([tuple(x) for x in args])
    raise ValueError(kind)


def ref_plan(spec):
    reps = [rt.Replica(*r) for r in spec["replicas"]]
    gears = []
    for g in spec["gears"]:
        gears.append(rt.Gear(cascade=rt.Cascade(stages=tuple(g["stages"]),
                                                thresholds=tuple(g["thresholds"])),
                             min_queue_length=dict(g["min_q"]),
                             load_weights={m: dict(w) for m, w in g["weights"].items()}))
    return rt.GearPlan(placement=rt.Placement(reps), slo=rt.Slo.latency(400_000),
                       qps_max=spec["qps_max"], gears=tuple(gears))


def main():
    out = {}
    for name, case in gi.replay_cases().items():
        prof = rsynth.make_profiles(case["profiles"]["n_models"],
                                    tuple(case["profiles"]["cost_ratios"]))
        n, easy, vseed = case["val"]
        val = rsynth.make_validation(prof, n_samples=n, easy_fraction=easy, seed=vseed)
        trace = ref_trace(case["trace"])
        plan = ref_plan(case["plan"])
        cfg = reng.EngineConfig(seed=case["seed"], measure_period_us=case["period"],
                                alpha=case["alpha"], initial_gear_index=case["initial_gear"],
                                enable_ticks=case["ticks"])
        m = reng.run(plan, trace, val, prof, config=cfg)
        recs = m.per_request
        out[f"{name}_arrivals"] = trace.arrivals
        out[f"{name}_horizon"] = np.array(trace.duration_us)
        out[f"{name}_rec"] = np.array(
            [[r.request_id, r.arrival_us, r.completion_us, r.stages_executed, int(r.correct),
              r.gear_index] for r in recs], dtype=np.int64).reshape(-1, 6)
        out[f"{name}_win"] = np.array(
            [[w.end_us, w.first_stage_queue_len, w.gear_before, w.candidate_gear, w.gear_after,
              w.observed_range, w.completed, -1 if w.p95_us is None else w.p95_us]
             for w in m.windows], dtype=np.int64).reshape(-1, 8)
        out[f"{name}_winf"] = np.array(
            [[w.measured_qps, np.nan if w.accuracy is None else w.accuracy] for w in m.windows],
            dtype=np.float64).reshape(-1, 2)
        out[f"{name}_counts"] = np.array([m.arrivals, m.completed, m.backlogged,
                                          m.in_flight_at_horizon], dtype=np.int64)
        out[f"{name}_qlen"] = np.array([m.queue_len_at_horizon[r[0]]
                                        for r in case["plan"]["replicas"]], dtype=np.int64)
        out[f"{name}_batches"] = np.array(json.dumps(
            {k: {str(b): c for b, c in v.items()} for k, v in m.per_model_batches.items()}))
        print(name, "arrivals", m.arrivals, "completed", m.completed, "windows", len(m.windows),
              "gears seen", sorted({r.gear_index for r in recs}))
    np.savez_compressed(HERE / "replay.npz", **out)
    man = json.loads((HERE / "MANIFEST.json").read_text())
    man["replay.npz"] = ("gearserve.engine.run (virtual clock) on golden_inputs.replay_cases(): "
                         "records, windows, counters, queues, batch histograms")
    (HERE / "MANIFEST.json").write_text(json.dumps(man, indent=1) + "\n")


if __name__ == "__main__":
    main()
