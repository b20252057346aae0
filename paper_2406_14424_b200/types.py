"""Domain types at the hot path's boundary.

Mirrors the subset of /root/reference/pkg/src/gearserve/types.py the cascade
API consumes: ModelProfile (:23-94), ProfileSet (:97-140), ModelOutput /
ValidationRecord / ValidationSet (:143-188) and Cascade (:191-221).  Same
field names, invariants and ValueError behaviour, so reference callers can
pass the same objects.  Two additions serve the B200 path:

* ValidationArrays — a columnar validation set (certainty / correct matrices,
  or raw per-model score rows) for 1M-sample workloads where building
  Python record objects would dominate.
* the per-set matrix cache also holds the device-resident copies.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

US_PER_S = 1_000_000


def _require(cond: bool, msg: str) -> None:
    if not cond:
        raise ValueError(msg)


@dataclass(frozen=True)
class ModelProfile:
    """Memory footprint and batch-latency table (batch -> total µs) of one
    model; batch 1 must be profiled, totals non-decreasing, per-sample
    latency non-increasing (reference types.py:23-60)."""

    model_id: str
    memory_bytes: int
    runtime_table: dict[int, int]

    def __post_init__(self) -> None:
        mid = self.model_id
        _require(isinstance(mid, str) and mid != "", "model_id must be a non-empty string")
        _require(isinstance(self.memory_bytes, int) and self.memory_bytes > 0,
                 f"{mid}: memory_bytes must be a positive integer")
        _require(len(self.runtime_table) > 0, f"{mid}: runtime_table is empty")
        for b, lat in self.runtime_table.items():
            _require(isinstance(b, int) and b >= 1,
                     f"{mid}: batch sizes must be integers >= 1, got {b!r}")
            _require(isinstance(lat, int) and lat > 0,
                     f"{mid}: latency for batch {b} must be a positive integer, got {lat!r}")
        _require(1 in self.runtime_table, f"{mid}: runtime_table must include batch size 1")
        batches = sorted(self.runtime_table)
        lats = [self.runtime_table[b] for b in batches]
        for (b0, l0), (b1, l1) in zip(zip(batches, lats), zip(batches[1:], lats[1:])):
            _require(l1 >= l0, f"{mid}: total latency decreases from batch {b0} to {b1}")
            _require(l1 * b0 <= l0 * b1,
                     f"{mid}: per-sample latency increases from batch {b0} to {b1}")
        object.__setattr__(self, "_batches", tuple(batches))
        object.__setattr__(self, "_latencies", tuple(lats))

    @property
    def profiled_batches(self) -> tuple[int, ...]:
        return self._batches  # type: ignore[attr-defined]

    @property
    def max_profiled_batch(self) -> int:
        return self._batches[-1]  # type: ignore[attr-defined]

    def runtime_us(self, batch: int) -> int:
        """Exact at profiled sizes, linear in between, error above the max."""
        _require(isinstance(batch, int) and batch >= 1,
                 f"{self.model_id}: batch must be an integer >= 1, got {batch!r}")
        lat = self.runtime_table.get(batch)
        if lat is not None:
            return lat
        batches, lats = self._batches, self._latencies  # type: ignore[attr-defined]
        if batch > batches[-1]:
            raise ValueError(
                f"{self.model_id}: batch {batch} exceeds max profiled batch {batches[-1]}")
        hi = next(i for i, b in enumerate(batches) if b >= batch)
        b0, b1, l0, l1 = batches[hi - 1], batches[hi], lats[hi - 1], lats[hi]
        return int(round(l0 + (l1 - l0) * (batch - b0) / (b1 - b0)))

    def per_sample_us(self, batch: int) -> float:
        return self.runtime_us(batch) / batch


class ProfileSet:
    """Ordered model profiles; insertion order is the canonical column order
    of every certainty/correct matrix (reference types.py:97-140)."""

    def __init__(self, models: list[ModelProfile]):
        by_id: dict[str, ModelProfile] = {}
        for m in models:
            _require(m.model_id not in by_id, f"duplicate model id {m.model_id!r}")
            by_id[m.model_id] = m
        _require(len(by_id) > 0, "profile set is empty")
        self._models = by_id
        self._order = tuple(by_id)
        self._index = {mid: i for i, mid in enumerate(self._order)}

    @property
    def model_ids(self) -> tuple[str, ...]:
        return self._order

    def __len__(self) -> int:
        return len(self._order)

    def __contains__(self, model_id: str) -> bool:
        return model_id in self._models

    def __getitem__(self, model_id: str) -> ModelProfile:
        try:
            return self._models[model_id]
        except KeyError:
            raise KeyError(f"unknown model id {model_id!r}") from None

    def __iter__(self):
        return iter(self._models.values())

    def index(self, model_id: str) -> int:
        return self._index[model_id]

    def runtime_us(self, model_id: str, batch: int) -> int:
        return self[model_id].runtime_us(batch)

    def cost1(self) -> np.ndarray:
        """Batch-1 runtimes in column order, f64 (reference cascades.py:92-93)."""
        return np.array([self._models[m].runtime_table[1] for m in self._order],
                        dtype=np.float64)

    def __eq__(self, other) -> bool:
        return isinstance(other, ProfileSet) and self._models == other._models

    def __repr__(self) -> str:
        return f"ProfileSet({list(self._order)!r})"


@dataclass(frozen=True)
class ModelOutput:
    """Recorded scores and correctness of one model on one sample."""

    scores: tuple[float, ...]
    correct: bool

    def __post_init__(self) -> None:
        _require(len(self.scores) >= 1, "scores must be non-empty")


@dataclass(frozen=True)
class ValidationRecord:
    sample_id: int
    outputs: dict[str, ModelOutput]


class ValidationSet:
    """Per-sample recorded outputs of every model (reference types.py:160-188).
    Caches derived matrices per model ordering (cascades.matrices)."""

    def __init__(self, records: list[ValidationRecord]):
        _require(len(records) > 0, "validation set is empty")
        keys = frozenset(records[0].outputs)
        _require(len(keys) > 0, "validation records cover no models")
        seen: set[int] = set()
        for r in records:
            _require(isinstance(r.sample_id, int) and r.sample_id >= 0,
                     f"sample_id must be a non-negative integer, got {r.sample_id!r}")
            _require(r.sample_id not in seen, f"duplicate sample_id {r.sample_id}")
            seen.add(r.sample_id)
            _require(frozenset(r.outputs) == keys,
                     f"sample {r.sample_id} covers models {sorted(r.outputs)}, "
                     f"expected {sorted(keys)}")
        self.records = list(records)
        self.model_ids = keys
        self._matrix_cache: dict = {}

    def __len__(self) -> int:
        return len(self.records)

    def __eq__(self, other) -> bool:
        return isinstance(other, ValidationSet) and self.records == other.records


class ValidationArrays:
    """Columnar validation set: for each model either a certainty column or a
    score matrix [n, n_cls] (f32 / f64 / bf16, numpy or torch), plus a
    correctness column.  Accepted wherever a ValidationSet is."""

    def __init__(self, model_ids, *, certainty=None, scores=None, correct=None, row_len=None,
                 sample_id=None):
        self.model_ids_ordered = tuple(model_ids)
        _require(len(self.model_ids_ordered) > 0, "validation covers no models")
        _require(len(set(self.model_ids_ordered)) == len(self.model_ids_ordered),
                 "duplicate model ids")
        _require(correct is not None, "correct is required")
        _require((certainty is None) != (scores is None),
                 "give exactly one of certainty= or scores=")
        self.certainty = certainty      # [n, M] or None
        self.scores = scores            # dict model_id -> [n, n_cls] or None
        self.correct = correct          # [n, M] u8 / bool
        self.row_len = row_len          # dict model_id -> [n] int (ragged score rows) or None
        self.sample_id = sample_id      # [n] int64 or None
        n = int(correct.shape[0])
        _require(n > 0, "validation set is empty")
        _require(tuple(correct.shape) == (n, len(self.model_ids_ordered)),
                 "correct must be [n_records, n_models]")
        if certainty is not None:
            _require(tuple(certainty.shape) == tuple(correct.shape),
                     "certainty and correct shapes differ")
        else:
            _require(set(scores) == set(self.model_ids_ordered), "scores must cover every model")
            for mid in self.model_ids_ordered:
                _require(scores[mid].ndim == 2 and int(scores[mid].shape[0]) == n,
                         f"{mid}: scores must be [n_records, n_cls]")
        self._n = n
        self.model_ids = frozenset(self.model_ids_ordered)
        self._matrix_cache: dict = {}

    def __len__(self) -> int:
        return self._n


@dataclass(frozen=True)
class Cascade:
    """Models cheap to expensive; a sample stops at stage i when its
    certainty reaches thresholds[i]; the final stage always stops
    (reference types.py:191-221)."""

    stages: tuple[str, ...]
    thresholds: tuple[float, ...]

    def __post_init__(self) -> None:
        _require(len(self.stages) >= 1, "cascade must have at least one stage")
        _require(len(set(self.stages)) == len(self.stages),
                 f"cascade repeats a model: {self.stages}")
        _require(len(self.thresholds) == len(self.stages) - 1,
                 f"cascade with {len(self.stages)} stages needs "
                 f"{len(self.stages) - 1} thresholds, got {len(self.thresholds)}")
        for t in self.thresholds:
            _require(t >= 0.0, f"thresholds must be >= 0, got {t}")

    @property
    def n_stages(self) -> int:
        return len(self.stages)

    def describe(self) -> str:
        parts = [f"{m}(>{self.thresholds[i]:g})" if i < len(self.thresholds) else m
                 for i, m in enumerate(self.stages)]
        return " -> ".join(parts)


# ---------------------------------------------------------------- serving --
# The plan / trace types the replay engine (replay.py, csrc/gs_engine.cu)
# consumes: reference types.py:232-469 (Replica, Placement, Gear, GearPlan,
# WorkloadTrace), reduced to the fields the event loop reads.  Reference
# objects of these classes are accepted as well (same attribute names).

@dataclass(frozen=True)
class Replica:
    replica_id: str
    model_id: str
    device_id: str


class Placement:
    """Model replicas on devices, in placement order (reference :247-306)."""

    def __init__(self, replicas):
        ids = [r.replica_id for r in replicas]
        _require(len(set(ids)) == len(ids), "duplicate replica id")
        pairs = [(r.model_id, r.device_id) for r in replicas]
        _require(len(set(pairs)) == len(pairs), "a model is placed twice on one device")
        self.replicas = tuple(replicas)

    def replicas_of(self, model_id: str):
        return tuple(r for r in self.replicas if r.model_id == model_id)

    def __len__(self) -> int:
        return len(self.replicas)


@dataclass(frozen=True)
class Gear:
    """Cascade, per-replica minimum batch (queue length) and per-model load
    split over replicas (reference :309-346)."""

    cascade: Cascade
    min_queue_length: dict
    load_weights: dict


@dataclass(frozen=True)
class GearPlan:
    """One gear per QPS range; range i covers [i, i+1) * qps_max / n_ranges,
    clamped to the top range (reference :376-410)."""

    placement: Placement
    slo: object
    qps_max: float
    gears: tuple

    @property
    def n_ranges(self) -> int:
        return len(self.gears)

    def range_for_qps(self, qps: float) -> int:
        _require(qps >= 0, f"qps must be >= 0, got {qps}")
        return min(int(np.floor(qps * self.n_ranges / self.qps_max)), self.n_ranges - 1)


class WorkloadTrace:
    """Non-decreasing integer-µs arrival times; the horizon defaults to the
    end of the last second holding an arrival (reference :433-469)."""

    def __init__(self, arrivals, duration_us: int | None = None):
        arrivals = np.asarray(arrivals, dtype=np.int64)
        if arrivals.size:
            _require(int(arrivals.min()) >= 0, "arrival times must be >= 0")
            _require(bool(np.all(np.diff(arrivals) >= 0)), "arrival times must be non-decreasing")
        if duration_us is None:
            duration_us = 0 if arrivals.size == 0 else (int(arrivals[-1]) // US_PER_S + 1) * US_PER_S
        else:
            _require(arrivals.size == 0 or int(arrivals[-1]) < duration_us,
                     "duration_us must exceed the last arrival")
        self.arrivals = arrivals
        self.duration_us = int(duration_us)

    def __len__(self) -> int:
        return int(self.arrivals.size)
