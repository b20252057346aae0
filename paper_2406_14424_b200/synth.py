"""Synthetic workloads for the hot path, vectorised.

make_profiles / make_validation_arrays restate gearserve.synth
(/root/reference/pkg/src/gearserve/synth.py:29-111) without building Python
record objects: the same numpy Generator draws in the same order, so the
certainty / correct matrices equal the reference's bit for bit
(tests/golden/synth.npz pins this), at 1M-sample scale in a fraction of a
second.  Tier semantics: tier 0 is easy (every model confident and
correct); tier t > 0 is answered correctly only by models with index >= t,
and a wrong model is unconfident; scores are (0.5 + c/2, 0.5 - c/2).

imagenet_logits builds the 1000-class config-3 workload on the device
(there is no reference generator for it).
"""

from __future__ import annotations

import numpy as np
import torch

from .types import ModelProfile, ProfileSet, ValidationArrays

DEFAULT_COST_RATIOS = (1.0, 4.0, 16.0)
DEFAULT_BATCHES = (1, 2, 4, 8)


def make_profiles(n_models: int = 3, cost_ratios=DEFAULT_COST_RATIOS,
                  base_runtime_us: int = 2_000, base_memory_bytes: int = 2_000_000_000,
                  memory_ratios=None, batches=DEFAULT_BATCHES,
                  batching_exponent: float = 0.7) -> ProfileSet:
    """Models m0..m{k-1}, cheapest first (reference synth.py:33-62)."""
    if n_models < 1:
        raise ValueError(f"n_models must be >= 1, got {n_models}")
    if len(cost_ratios) != n_models:
        raise ValueError(f"need {n_models} cost ratios, got {len(cost_ratios)}")
    if any(r <= 0 for r in cost_ratios):
        raise ValueError("cost ratios must be positive")
    if list(cost_ratios) != sorted(cost_ratios):
        raise ValueError("cost ratios must be non-decreasing")
    if not (0 < batching_exponent <= 1):
        raise ValueError("batching exponent must be in (0, 1]")
    memory_ratios = memory_ratios if memory_ratios is not None else cost_ratios
    if len(memory_ratios) != n_models:
        raise ValueError(f"need {n_models} memory ratios, got {len(memory_ratios)}")
    models = []
    for j in range(n_models):
        r1 = base_runtime_us * cost_ratios[j]
        table = {b: int(round(r1 * b ** batching_exponent)) for b in sorted(batches)}
        models.append(ModelProfile(model_id=f"m{j}",
                                   memory_bytes=int(round(base_memory_bytes * memory_ratios[j])),
                                   runtime_table=table))
    return ProfileSet(models)


def tier_pattern(n_samples: int, easy_fraction: float, n_tiers: int) -> np.ndarray:
    """Bresenham-spread difficulty tiers (reference synth.py:65-75)."""
    tiers = np.zeros(n_samples, dtype=np.int64)
    if easy_fraction >= 1.0:
        return tiers
    i = np.arange(n_samples, dtype=np.int64)
    hard = np.flatnonzero(((i + 1) * easy_fraction).astype(np.int64)
                          == (i * easy_fraction).astype(np.int64))
    tiers[hard] = 1 + np.arange(hard.size) % max(1, n_tiers)
    return tiers


def validation_matrices(n_models: int, n_samples: int, easy_fraction: float = 0.8,
                        seed: int = 0, confident_range=(0.6, 0.95), unsure_range=(0.0, 0.3),
                        shuffle: bool = False, return_scores: bool = False):
    """(certainty [n, M] f64, correct [n, M] u8[, scores [M][n, 2] f64]) with the
    reference make_validation semantics and RNG stream."""
    if not 0.0 <= easy_fraction <= 1.0:
        raise ValueError(f"easy_fraction must be in [0, 1], got {easy_fraction}")
    if n_samples < 1:
        raise ValueError(f"n_samples must be >= 1, got {n_samples}")
    if not confident_range[0] > unsure_range[1]:
        raise ValueError("confident range must sit strictly above unsure range")
    tiers = tier_pattern(n_samples, easy_fraction, max(1, n_models - 1))
    rng = np.random.default_rng(seed)
    if shuffle:
        tiers = rng.permutation(tiers)
    correct = tiers[:, None] <= np.arange(n_models)[None, :]
    lo = np.where(correct, confident_range[0], unsure_range[0])
    hi = np.where(correct, confident_range[1], unsure_range[1])
    c = rng.uniform(lo, hi)                      # C order = (sample, model) loop order
    top = 0.5 + c / 2
    second = 0.5 - c / 2
    cert = top - second                          # cascades.certainty on the 2-score tuple
    out = (np.ascontiguousarray(cert), correct.astype(np.uint8))
    if return_scores:
        out = out + (np.stack([top, second], axis=-1).transpose(1, 0, 2),)
    return out


def make_validation_arrays(profiles: ProfileSet, n_samples: int = 500,
                           easy_fraction: float = 0.8, seed: int = 0,
                           confident_range=(0.6, 0.95), unsure_range=(0.0, 0.3),
                           shuffle: bool = False) -> ValidationArrays:
    """Columnar make_validation (reference synth.py:78-111)."""
    cert, corr = validation_matrices(len(profiles), n_samples, easy_fraction, seed,
                                     confident_range, unsure_range, shuffle)
    return ValidationArrays(profiles.model_ids, certainty=cert, correct=corr)


def binary_logit_arrays(profiles: ProfileSet, n_samples: int, easy_fraction: float = 0.8,
                        seed: int = 0, dtype=np.float32) -> ValidationArrays:
    """Config-2 shape: per-model binary score heads [n, 2] in `dtype`
    (reference semantics; certainty is then the margin of the stored
    values, computed on the device)."""
    _, corr, scores = validation_matrices(len(profiles), n_samples, easy_fraction, seed,
                                          return_scores=True)
    return ValidationArrays(profiles.model_ids,
                            scores={m: np.ascontiguousarray(scores[j].astype(dtype))
                                    for j, m in enumerate(profiles.model_ids)},
                            correct=corr)


def imagenet_logits(n_samples: int, n_cls: int = 1000, n_models: int = 3, seed: int = 0,
                    dtype: torch.dtype = torch.float32, device=None):
    """Config-3 shape on the device: per model [n, n_cls] logits ~ N(0, 1)
    with the label's logit boosted on rows the model gets right; a model of
    index j is right on tiers <= j (same tier scheme as make_validation)."""
    device = device or torch.device("cuda")
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    tiers = torch.from_numpy(tier_pattern(n_samples, 0.8, max(1, n_models - 1))).to(device)
    labels = torch.randint(0, n_cls, (n_samples,), generator=g, device=device)
    rows = torch.arange(n_samples, device=device)
    out, correct = [], []
    for j in range(n_models):
        x = torch.randn((n_samples, n_cls), generator=g, device=device, dtype=torch.float32)
        right = tiers <= j
        boost = torch.where(right, 4.0 + 2.0 * torch.rand(n_samples, generator=g, device=device),
                            torch.zeros(n_samples, device=device))
        x[rows, labels] += boost
        out.append(x.to(dtype))
        correct.append(right.to(torch.uint8))
    return out, torch.stack(correct, dim=1), labels


def kernels_bench_problem(n_records: int = 4000, n_models: int = 6, n_cascades: int = 200,
                          seed: int = 0):
    """The reference's own operator benchmark problem
    (pkg/benchmarks/bench_kernels.py:25-49, the published 5.3 ms numba /
    17.0 ms numpy point at records=4000 models=6 cascades=200): the same
    Generator draws in the same order, returned as evaluate_encoded's
    positional arguments (certainty, correct, stage_model, thresholds,
    n_stages, cost1)."""
    rng = np.random.default_rng(seed)
    mids = [f"m{j}" for j in range(n_models)]
    cost1 = np.array([int(rng.integers(1_000, 60_000)) for _ in mids], dtype=np.float64)
    index = {m: j for j, m in enumerate(mids)}
    stages_list, thr_list = [], []
    for _ in range(n_cascades):
        k = int(rng.integers(1, n_models + 1))
        stages_list.append(tuple(rng.permutation(mids)[:k]))
        thr_list.append(tuple(float(x) for x in rng.random(k - 1)))
    max_len = max(len(s) for s in stages_list)
    stage_model = np.full((n_cascades, max_len), -1, dtype=np.int32)
    thresholds = np.zeros((n_cascades, max_len))
    n_stages = np.zeros(n_cascades, dtype=np.int32)
    for ci, (s, t) in enumerate(zip(stages_list, thr_list)):
        n_stages[ci] = len(s)
        stage_model[ci, : len(s)] = [index[m] for m in s]
        thresholds[ci, : len(t)] = t
    certainty = rng.random((n_records, n_models))
    correct = (rng.random((n_records, n_models)) < 0.7).astype(np.uint8)
    return certainty, correct, stage_model, thresholds, n_stages, cost1


def bursty_counts(seconds: int, seed: int = 0, base: float = 100.0, sigma: float = 0.7):
    """Per-second request counts of an Azure-like bursty series (lognormal
    levels, default_rng(seed)); scale with replay.scale_trace."""
    rng = np.random.default_rng(seed)
    return np.rint(base * rng.lognormal(0.0, sigma, seconds)).astype(np.int64) + 1


def trace_from_counts(counts):
    """Arrivals at the start of each second, counts[s] of them (the input
    scale_trace reads per-second counts from)."""
    from .types import WorkloadTrace
    counts = np.asarray(counts, dtype=np.int64)
    return WorkloadTrace(np.repeat(np.arange(counts.size, dtype=np.int64) * 1_000_000, counts))


def constant_rate_trace(qps: float, seconds: float):
    """Evenly spaced arrivals (reference synth.constant_rate_trace :121-133)."""
    from .types import WorkloadTrace
    if qps <= 0 or seconds <= 0:
        raise ValueError("qps and seconds must be positive")
    n = int(round(qps * seconds))
    if n == 0:
        raise ValueError(f"qps {qps} over {seconds}s yields no arrivals")
    arrivals = np.floor(np.arange(n, dtype=np.float64) * (1_000_000 / qps)).astype(np.int64)
    duration = int(round(seconds * 1_000_000))
    if int(arrivals[-1]) >= duration:
        duration = (int(arrivals[-1]) // 1_000_000 + 1) * 1_000_000
    return WorkloadTrace(arrivals, duration_us=duration)


def step_trace(steps):
    """Constant-rate segments [(qps, seconds), ...] back to back, qps 0 =
    silence (reference synth.step_trace :135-154)."""
    from .types import WorkloadTrace
    if not steps:
        raise ValueError("step trace needs at least one segment")
    parts, offset = [], 0
    for qps, seconds in steps:
        if seconds <= 0:
            raise ValueError(f"segment duration must be positive, got {seconds}")
        if qps < 0:
            raise ValueError(f"segment qps must be >= 0, got {qps}")
        if qps > 0:
            parts.append(constant_rate_trace(qps, seconds).arrivals + offset)
        offset += int(round(seconds * 1_000_000))
    if not parts:
        raise ValueError("step trace has no arrivals")
    return WorkloadTrace(np.concatenate(parts), duration_us=offset)


def replica_group_plan(qps_max: float = 950.0, prefix: str = ""):
    """Config 5's replica group (one per GPU): a Sentiment-140-shaped 4-model
    cascade (make_profiles(4, cost ratios 1:4:16:64, 1 ms base)) on four
    devices, and one gear per QPS quarter, from the full cascade at low load
    to the cheapest model alone at the top range (the gear switching the
    engine's tick applies).  Returns (profiles, plan)."""
    from .types import Cascade, Gear, GearPlan, Placement, Replica
    prof = make_profiles(n_models=4, cost_ratios=(1.0, 4.0, 16.0, 64.0), base_runtime_us=1_000)
    d = [f"{prefix}d{i}" for i in range(4)]
    reps = [Replica(f"m0@{d[0]}", "m0", d[0]), Replica(f"m0@{d[1]}", "m0", d[1]),
            Replica(f"m1@{d[1]}", "m1", d[1]), Replica(f"m1@{d[2]}", "m1", d[2]),
            Replica(f"m2@{d[2]}", "m2", d[2]), Replica(f"m3@{d[3]}", "m3", d[3])]
    w0 = {f"m0@{d[0]}": 2.0, f"m0@{d[1]}": 1.0}
    w1 = {f"m1@{d[1]}": 1.0, f"m1@{d[2]}": 1.0}
    gears = (
        Gear(Cascade(("m0", "m1", "m2", "m3"), (0.62, 0.7, 0.75)), {f"m0@{d[0]}": 2},
             {"m0": w0, "m1": w1, "m2": {f"m2@{d[2]}": 1.0}, "m3": {f"m3@{d[3]}": 1.0}}),
        Gear(Cascade(("m0", "m1", "m2"), (0.66, 0.72)), {f"m0@{d[0]}": 4},
             {"m0": w0, "m1": w1, "m2": {f"m2@{d[2]}": 1.0}}),
        Gear(Cascade(("m0", "m1"), (0.7,)), {f"m0@{d[0]}": 8, f"m0@{d[1]}": 4},
             {"m0": w0, "m1": w1}),
        Gear(Cascade(("m0",), ()), {f"m0@{d[0]}": 8, f"m0@{d[1]}": 8}, {"m0": w0}),
    )
    return prof, GearPlan(placement=Placement(reps), slo=None, qps_max=qps_max, gears=gears)
