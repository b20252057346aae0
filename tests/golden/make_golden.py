"""Capture golden vectors from the reference itself (run where the reference
is importable; the GPU box never reads /root/reference).

    GEARSERVE_REF_SRC=/root/reference/pkg/src python tests/golden/make_golden.py

Inputs that numpy can regenerate deterministically (default_rng streams)
are stored as seeds plus a checksum; reference outputs are stored in full.
Every fixture records which reference function produced it.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF_SRC = os.environ.get("GEARSERVE_REF_SRC", "/root/reference/pkg/src")
sys.path.insert(0, REF_SRC)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from gearserve import cascades as rc  # noqa: E402
from gearserve import engine as reng  # noqa: E402
from gearserve import kernels as rk  # noqa: E402
from gearserve import synth as rsynth  # noqa: E402
from gearserve import types as rt  # noqa: E402

sys.path.insert(0, str(HERE.parent))
import golden_inputs as gi  # noqa: E402


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def kernels_fixtures(meta):
    """test_kernels._random_problem (pkg/tests/test_kernels.py:7-19) x5 with
    default_rng(12345), the bench_kernels default problem
    (pkg/benchmarks/bench_kernels.py:25-49), and the known-answer cases."""
    out = {}
    rng = np.random.default_rng(12345)
    for t in range(5):
        args = gi.random_problem(rng)
        acc, cost, frac = rk._evaluate_numba(*args)
        out[f"rp{t}_sha"] = np.frombuffer(bytes.fromhex(sha(*args)), dtype=np.uint8)
        out[f"rp{t}_acc"], out[f"rp{t}_cost"], out[f"rp{t}_frac"] = acc, cost, frac
    args = gi.bench_problem(4000, 6, 200, 0)
    acc, cost, frac = rk._evaluate_numba(*args)
    out["bench_sha"] = np.frombuffer(bytes.fromhex(sha(*args)), dtype=np.uint8)
    out["bench_acc"], out["bench_cost"], out["bench_frac"] = acc, cost, frac
    np.savez_compressed(HERE / "kernels.npz", **out)
    meta["kernels.npz"] = "gearserve.kernels._evaluate_numba on test_kernels/bench_kernels problems"


def c1_fixtures(meta):
    """test_acceptance C1 fixtures (pkg/tests/test_acceptance.py:115-151):
    ragged score tuples -> reference matrices + evaluate_cascades."""
    out = {}
    for i, fx in enumerate(gi.c1_fixtures()):
        profiles = rt.ProfileSet([rt.ModelProfile(m, 1_000_000, {1: c})
                                  for m, c in zip(fx["mids"], fx["cost1"])])
        recs = []
        for r in range(fx["n_rec"]):
            outs = {m: rt.ModelOutput(scores=tuple(float(x) for x in
                                                   fx["scores"][r * len(fx["mids"]) + j,
                                                                : fx["lens"][r * len(fx["mids"]) + j]]),
                                      correct=bool(fx["correct"][r, j]))
                    for j, m in enumerate(fx["mids"])}
            recs.append(rt.ValidationRecord(sample_id=r, outputs=outs))
        val = rt.ValidationSet(recs)
        cert, corr = rc.matrices(val, profiles)
        cascs = [rt.Cascade(stages=tuple(s), thresholds=tuple(t)) for s, t in fx["cascades"]]
        evs = rc.evaluate_cascades(cascs, val, profiles)
        out[f"f{i}_cert"] = cert
        out[f"f{i}_corr"] = corr
        out[f"f{i}_acc"] = np.array([e.accuracy for e in evs])
        out[f"f{i}_cost"] = np.array([e.mean_cost for e in evs])
        width = max(len(s) for s, _ in fx["cascades"])
        ff = np.zeros((len(evs), width))
        for k, (e, (s, _)) in enumerate(zip(evs, fx["cascades"])):
            ff[k, : len(s)] = [e.forward_fraction[m] for m in s]
        out[f"f{i}_frac"] = ff
    np.savez_compressed(HERE / "c1.npz", **out)
    meta["c1.npz"] = "gearserve.cascades.matrices + evaluate_cascades on the C1 acceptance fixtures"


def config1_fixture(meta):
    """Config 1: synth.make_profiles() + make_validation(n=10_000, seed=0),
    100-level grids, full grid product scored by the reference numba walk."""
    profiles = rsynth.make_profiles()
    val = rsynth.make_validation(profiles, n_samples=10_000, easy_fraction=0.8, seed=0)
    cert, corr = rc.matrices(val, profiles)
    grid = rc.build_threshold_grid(val, profiles, levels=100)
    grids = [np.array(grid.per_model[m]) for m in profiles.model_ids]
    sm, thr, ns = gi.grid_configs_py(grids)
    cost1 = np.array([profiles[m].runtime_table[1] for m in profiles.model_ids], dtype=np.float64)
    acc, cost, frac = rk._evaluate_numba(cert, corr, sm, thr, ns, cost1)
    np.savez_compressed(HERE / "config1.npz", cert_sha=np.frombuffer(bytes.fromhex(sha(cert, corr)), np.uint8),
                        grid0=grids[0], grid1=grids[1], grid2=grids[2], cost1=cost1,
                        acc=acc, cost=cost, frac=frac)
    meta["config1.npz"] = ("synth.make_validation(make_profiles(), 10000, 0.8, seed=0); "
                           "build_threshold_grid(levels=100); numba walk over the full product")


def certainty_fixture(meta):
    """cascades.certainty on ragged tuples (duplicates, negatives,
    singletons) and on f32 1000-class logits promoted to f64."""
    rows, lens = gi.certainty_tuples()
    ref = np.array([rc.certainty(tuple(float(x) for x in rows[i, : lens[i]]))
                    for i in range(rows.shape[0])])
    logits = gi.logits_f32(seed=3, n=256, n_cls=1000)
    ref_logits = np.array([rc.certainty(tuple(float(x) for x in row)) for row in logits])
    np.savez_compressed(HERE / "certainty.npz", tuples=ref, logits=ref_logits,
                        logits_sha=np.frombuffer(bytes.fromhex(sha(logits)), np.uint8))
    meta["certainty.npz"] = "gearserve.cascades.certainty on ragged tuples and f32 logits"


def pareto_fixture(meta):
    out = {}
    for t, (acc, cost) in enumerate(gi.pareto_cases()):
        cas = [rt.Cascade(stages=(f"m{i}",), thresholds=()) for i in range(len(acc))]
        evs = [(c, rc.CascadeEval(accuracy=float(a), mean_cost=float(b), forward_fraction={}))
               for c, a, b in zip(cas, acc, cost)]
        kept = rc.pareto_filter(evs)
        ids = {id(c) for c, _ in kept}
        out[f"p{t}_keep"] = np.array([id(c) in ids for c in cas], dtype=bool)
    np.savez_compressed(HERE / "pareto.npz", **out)
    meta["pareto.npz"] = "gearserve.cascades.pareto_filter on random points with exact ties"


def grid_and_sampler_fixture(meta):
    """build_threshold_grid + sample_cascades on the conftest fixtures."""
    profiles = rt.ProfileSet([
        rt.ModelProfile("small", 4_000_000_000, {1: 5_000, 2: 8_000, 4: 12_000}),
        rt.ModelProfile("large", 10_000_000_000, {1: 20_000, 2: 32_000, 4: 48_000})])
    recs = []
    for i in range(100):
        hard = (i % 5) == 4
        small = rt.ModelOutput(scores=(0.5, 0.45), correct=False) if hard else \
            rt.ModelOutput(scores=(0.9, 0.05), correct=True)
        large = rt.ModelOutput(scores=(0.95,), correct=(i % 20) != 19)
        recs.append(rt.ValidationRecord(sample_id=i, outputs={"small": small, "large": large}))
    val = rt.ValidationSet(recs)
    out = {}
    for levels in (2, 4, 10):
        g = rc.build_threshold_grid(val, profiles, levels=levels)
        for m in profiles.model_ids:
            out[f"grid_{levels}_{m}"] = np.array(g.per_model[m])
    g = rc.build_threshold_grid(val, profiles)
    for seed in (0, 1, 7):
        cs = rc.sample_cascades(profiles, g, n_samples=100, rng_seed=seed)
        out[f"sample_{seed}"] = np.array(json.dumps([[list(c.stages), list(c.thresholds)]
                                                     for c in cs]))
    # 3-model synth profiles, 400 samples (acceptance fixtures)
    p3 = rsynth.make_profiles()
    v3 = rsynth.make_validation(p3, n_samples=400, easy_fraction=0.8, seed=0)
    g3 = rc.build_threshold_grid(v3, p3, levels=10)
    for m in p3.model_ids:
        out[f"synth_grid_{m}"] = np.array(g3.per_model[m])
    cs = rc.sample_cascades(p3, g3, n_samples=2000, rng_seed=11)
    out["synth_sample"] = np.array(json.dumps([[list(c.stages), list(c.thresholds)] for c in cs]))
    np.savez_compressed(HERE / "grid_sampler.npz", **out)
    meta["grid_sampler.npz"] = "gearserve.cascades.build_threshold_grid + sample_cascades"


def synth_fixture(meta):
    """make_validation matrices for the vectorised generator (sha only)."""
    out = {}
    for n_models, n, ef, seed, shuffle in ((3, 1000, 0.8, 0, False), (4, 2000, 0.7, 5, True),
                                           (2, 333, 0.5, 1, False)):
        ratios = tuple(float(4 ** j) for j in range(n_models))
        p = rsynth.make_profiles(n_models=n_models, cost_ratios=ratios)
        v = rsynth.make_validation(p, n_samples=n, easy_fraction=ef, seed=seed, shuffle=shuffle)
        cert, corr = rc.matrices(v, p)
        key = f"{n_models}_{n}_{ef}_{seed}_{int(shuffle)}"
        out[key] = np.frombuffer(bytes.fromhex(sha(cert, corr)), np.uint8)
    np.savez_compressed(HERE / "synth.npz", **out)
    meta["synth.npz"] = "sha256 of gearserve.synth.make_validation matrices"


def engine_fixture(meta):
    """EngineState.finish_batch on random batches over multi-gear plans."""
    cases = gi.engine_cases()
    out = {}
    for t, case in enumerate(cases):
        profiles = rt.ProfileSet([rt.ModelProfile(m, 1_000_000, {1: 1000 * (j + 1), 8: 4000 * (j + 1)})
                                  for j, m in enumerate(case["mids"])])
        recs = []
        for r in range(case["n_rec"]):
            outs = {m: rt.ModelOutput(scores=(float(case["cert"][r, j]),),
                                      correct=bool(case["corr"][r, j]))
                    for j, m in enumerate(case["mids"])}
            recs.append(rt.ValidationRecord(sample_id=r, outputs=outs))
        val = rt.ValidationSet(recs)
        replicas = [rt.Replica(rid, m, d) for rid, m, d in case["replicas"]]
        pl = rt.Placement(replicas)
        gears = []
        for g in case["gears"]:
            lw = {m: {rid: w for rid, w in g["weights"][m].items()} for m in g["stages"]}
            gears.append(rt.Gear(cascade=rt.Cascade(stages=tuple(g["stages"]),
                                                    thresholds=tuple(g["thresholds"])),
                                 min_queue_length={rid: 1 for rid, _, _ in case["replicas"]},
                                 load_weights=lw))
        plan = rt.GearPlan(placement=pl, slo=rt.Slo.latency(1_000_000), qps_max=100.0,
                           gears=tuple(gears))
        comp = reng.CompiledPlan(plan, profiles, val)
        state = reng.EngineState(comp, reng.EngineConfig(seed=case["seed"]))
        items = [reng._Item(it["request_id"], it["row"], it["stage"], it["gear"], it["arrival_us"])
                 for it in case["items"]]
        touched = state.finish_batch(0, items, case["now"])
        done = [(r.request_id, int(r.correct), r.stages_executed, r.completion_us - r.arrival_us)
                for r in state.request_records]
        queues = [[(it.request_id, it.stage) for it in q] for q in state.queues]
        out[f"e{t}"] = np.array(json.dumps({"done": done, "queues": queues,
                                            "touched": sorted(touched),
                                            "rng_next": float(state.rng.random())}))
    np.savez_compressed(HERE / "engine.npz", **out)
    meta["engine.npz"] = "gearserve.engine.EngineState.finish_batch on random multi-gear batches"


INGEST_OK = """{"sample_id": 0, "models": {"a": {"scores": [0.1, 0.7, 0.2], "correct": true}, "b": {"scores": [0.5], "correct": false}}}

{"models": {"b": {"correct": 1, "scores": [1e-5, -2.5e+3]}, "a": {"scores": [3, 4], "correct": 0}}, "sample_id": 7, "extra": [1, {"x": null}, "s"]}
{"sample_id": 3.0, "models": {"a": {"scores": [NaN, 1.0], "correct": true, "note": "hi"}, "b": {"scores": [Infinity, -Infinity, 0.0], "correct": false}}}
   
{"sample_id": 12, "models": {"a": {"scores": [0.30000000000000004, "0.25"], "correct": false}, "b": {"scores": [5e-324, 1.7976931348623157e308], "correct": true}}}
"""

INGEST_BAD = {
    "missing_correct": '{"sample_id": 0, "models": {"a": {"scores": [1.0], "correct": true}}}\n'
                       '{"sample_id": 1, "models": {"a": {"scores": [1.0]}}}\n',
    "empty_scores": '{"sample_id": 0, "models": {"a": {"scores": [1.0], "correct": true}}}\n\n'
                    '{"sample_id": 1, "models": {"a": {"scores": [], "correct": true}}}\n',
    "not_json": '{"sample_id": 0, "models": {"a": {"scores": [1.0], "correct": true}}}\n{oops\n',
    "duplicate_id": '{"sample_id": 4, "models": {"a": {"scores": [1.0], "correct": true}}}\n'
                    '{"sample_id": 4, "models": {"a": {"scores": [2.0], "correct": true}}}\n',
    "model_mismatch": '{"sample_id": 0, "models": {"a": {"scores": [1.0], "correct": true}}}\n'
                      '{"sample_id": 1, "models": {"b": {"scores": [1.0], "correct": true}}}\n',
    "negative_id": '{"sample_id": -1, "models": {"a": {"scores": [1.0], "correct": true}}}\n',
    "bad_score": '{"sample_id": 0, "models": {"a": {"scores": ["x"], "correct": true}}}\n',
}


def ingest_fixture(meta):
    """gearserve.formats.load_validation (src/formats.py:75-97) on an
    edge-case JSONL (blank lines, key order, extra keys, NaN / Infinity,
    string scores, ragged and singleton score lists) and on malformed files
    (the reference's error: ValueError, with the line number when the
    reader names one)."""
    from gearserve import formats as rf
    ok = HERE / "ingest_ok.jsonl"
    ok.write_text(INGEST_OK)
    v = rf.load_validation(ok)
    recs = [{"sample_id": r.sample_id,
             "models": {m: {"scores": [repr(float(x)) for x in o.scores], "correct": o.correct}
                        for m, o in r.outputs.items()}} for r in v.records]
    bad = {}
    for name, text in INGEST_BAD.items():
        path = HERE / f"ingest_bad_{name}.jsonl"
        path.write_text(text)
        try:
            rf.load_validation(path)
            bad[name] = None
        except ValueError as e:
            msg = str(e)
            line = None
            if ": line " in msg:
                line = int(msg.split(": line ")[1].split(":")[0])
            bad[name] = {"line": line}
    (HERE / "ingest.json").write_text(json.dumps({"ok": recs, "bad": bad}, indent=1) + "\n")
    meta["ingest.json"] = ("gearserve.formats.load_validation on ingest_ok.jsonl and the "
                           "ingest_bad_*.jsonl files")


def main():
    meta = {"reference_src": REF_SRC, "numpy": np.__version__}
    kernels_fixtures(meta)
    c1_fixtures(meta)
    config1_fixture(meta)
    certainty_fixture(meta)
    pareto_fixture(meta)
    grid_and_sampler_fixture(meta)
    synth_fixture(meta)
    engine_fixture(meta)
    ingest_fixture(meta)
    (HERE / "MANIFEST.json").write_text(json.dumps(meta, indent=1) + "\n")
    print(json.dumps(meta, indent=1))


if __name__ == "__main__":
    main()
