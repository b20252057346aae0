"""Host side of the device replay (no GPU): the traces it replays equal the
reference's (scale_trace, constant/step traces, golden arrivals), and the
device PCG64 stream it relies on is numpy's (restated in oracle.Pcg64)."""

import numpy as np

import golden_inputs as gi
from conftest import golden
from oracle import oracle


def test_traces_match_the_reference_goldens():
    from replay_cases import build
    g = golden("replay.npz")
    for name, case in gi.replay_cases().items():
        _, _, trace, _, _ = build(case)
        assert np.array_equal(trace.arrivals, g[f"{name}_arrivals"]), name
        assert trace.duration_us == int(g[f"{name}_horizon"]), name


def test_split_round_robin():
    from paper_2406_14424_b200 import replay, synth
    t = replay.scale_trace(synth.trace_from_counts(synth.bursty_counts(30, 1)), 500.0)
    parts = replay.split_round_robin(t, 3)
    assert sum(len(p) for p in parts) == len(t)
    assert np.array_equal(np.sort(np.concatenate([p.arrivals for p in parts])), t.arrivals)


def test_pcg64_restatement_matches_numpy():
    """The draws gs_engine.cu reproduces: random(), integers(n) (Lemire, with
    the bit generator's buffered 32-bit half), interleaved."""
    for seed in range(4):
        a = np.random.default_rng(seed)
        b = oracle.Pcg64(seed)
        for t in range(3000):
            if t % 3 == 1:
                n = 1 + t % 9
                assert int(a.integers(n)) == b.integers(n)
            else:
                assert a.random() == b.random()
        assert b.state() == (a.bit_generator.state["state"]["state"],
                             a.bit_generator.state["has_uint32"],
                             a.bit_generator.state["uinteger"])


def test_sampler_restatement_matches_numpy_sampler():
    """oracle.sample_cascades_pcg (the algorithm gs_sampler.cu runs) equals
    the numpy sampler (the reference's stream), incl. 1- and 2-value grids
    (no draw / one-bit draws) and M = 1..6."""
    from paper_2406_14424_b200.cascades import ThresholdGrid, sample_cascades
    from paper_2406_14424_b200 import synth
    for M, lens, seed, n in ((3, (10, 10, 10), 0, 500), (1, (4,), 3, 20), (4, (1, 2, 7, 1), 5, 400),
                             (6, (3, 100, 1, 2, 50, 9), 9, 300)):
        prof = synth.make_profiles(n_models=M, cost_ratios=tuple(float(4 ** j) for j in range(M)))
        ids = prof.model_ids
        grid = ThresholdGrid({m: tuple(float(x) for x in np.arange(lens[j]) / 100.0)
                              for j, m in enumerate(ids)})
        want = sample_cascades(prof, grid, n, rng_seed=seed)
        got, _ = oracle.sample_cascades_pcg(lens, n, seed)  # cost order == column order here
        assert len(got) == len(want)
        for (ranks, gidx), c in zip(got, want):
            assert tuple(ids[r] for r in ranks) == c.stages
            assert tuple(grid.per_model[ids[r]][i] for r, i in zip(ranks, gidx)) == c.thresholds


def test_oracle_engine_matches_reference_goldens():
    """oracle.engine_run (the CPU checker of the device replay) equals the
    reference engine.run goldens on every scenario."""
    from replay_cases import build
    g = golden("replay.npz")
    for name, case in gi.replay_cases().items():
        prof, val, trace, plan, cfg = build(case)
        ids = list(prof.model_ids)
        cap = max(prof[m].max_profiled_batch for m in ids)
        runtime = [[0] + [prof[m].runtime_us(b) for b in range(1, cap + 1)] for m in ids]
        out = oracle.engine_run(plan, trace, val.certainty, val.correct, runtime,
                                [prof[m].max_profiled_batch for m in ids],
                                {m: j for j, m in enumerate(ids)}, seed=cfg.seed,
                                period_us=cfg.measure_period_us, alpha=cfg.alpha,
                                initial_gear=cfg.initial_gear_index, enable_ticks=cfg.enable_ticks)
        assert np.array_equal(out["records"], g[f"{name}_rec"]), name
        w = np.array([[x[0], x[2], x[3], x[4], x[5], x[4], x[6], x[7]] for x in out["windows"]],
                     dtype=np.int64).reshape(-1, 8)
        assert np.array_equal(w, g[f"{name}_win"]), name
        wf = np.array([[x[1], x[8]] for x in out["windows"]]).reshape(-1, 2)
        assert np.array_equal(wf, g[f"{name}_winf"], equal_nan=True), name
        assert out["queue_len"] == g[f"{name}_qlen"].tolist(), name
