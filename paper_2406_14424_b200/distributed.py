"""Multi-GPU gear-plan sweep: one process per GPU, configs partitioned per
rank, NCCL all-gather of the per-rank Pareto fronts.

The reference is single-process but declares cascade
evaluations safe for data-parallel evaluation.  Pareto
dominance is transitive, so the global front of the full config space is the
front of the union of the per-rank fronts; merging the gathered fronts with
the same exact reduction (gs_pareto_counts) gives the single-GPU answer, and
since rank r owns a contiguous config range below rank r+1's, concatenating
the per-rank fronts in rank order keeps ascending config order — the
reference's "input order" (cascades.py:116-129).

Front records travel as int64 triples (config index, correct count, cost as
raw f64 bits), so the exchange is bit-exact.
"""

from __future__ import annotations

import torch
import torch.distributed as dist


def shard_ranges(n_configs: int, world: int) -> list[tuple[int, int]]:
    """Contiguous, near-equal (begin, count) config ranges, rank order."""
    base, extra = divmod(n_configs, world)
    out, off = [], 0
    for r in range(world):
        n = base + (1 if r < extra else 0)
        out.append((off, n))
        off += n
    return out


def pack_front(idx: torch.Tensor, n_correct: torch.Tensor, mean_cost: torch.Tensor) -> torch.Tensor:
    """[k, 3] int64 records (index, correct count, cost bits)."""
    return torch.stack([idx.to(torch.int64), n_correct.to(torch.int64),
                        mean_cost.to(torch.float64).view(torch.int64)], dim=1).contiguous()


def unpack_front(rec: torch.Tensor):
    idx = rec[:, 0].contiguous()
    n_correct = rec[:, 1].to(torch.int32).contiguous()
    cost = rec[:, 2].contiguous().view(torch.float64)
    return idx, n_correct, cost


def all_gather_records(rec: torch.Tensor, group=None) -> torch.Tensor:
    """All-gather variable-length [k_r, 3] int64 blocks: sizes first, then
    payloads padded to the largest, concatenated in rank order."""
    world = dist.get_world_size(group)
    n = torch.tensor([rec.shape[0]], dtype=torch.int64, device=rec.device)
    sizes = [torch.empty_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    sizes = [int(s.item()) for s in sizes]
    width = max(max(sizes), 1)
    pad = torch.zeros((width, rec.shape[1]), dtype=rec.dtype, device=rec.device)
    pad[: rec.shape[0]] = rec
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    return torch.cat([b[:s] for b, s in zip(bufs, sizes)], dim=0)


def gather_fronts(idx: torch.Tensor, res, world: int, group=None) -> torch.Tensor:
    """Gather every rank's front records (index relative to its own range
    start in res.config_begin) to every rank."""
    local = idx - res.config_begin
    rec = pack_front(idx, res.n_correct[local], res.mean_cost[local])
    if world == 1:
        return rec
    return all_gather_records(rec, group)


def sharded_front(sweep, group=None):
    """Global Pareto front of a GridSweep whose table every rank has built:
    score this rank's config range, reduce it to its local front, all-gather,
    merge.  Returns (config indices ascending, correct counts, costs)."""
    from .gridsweep import pareto_counts
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    begin, count = shard_ranges(sweep.n_configs, world)[rank]
    res = sweep.evaluate(begin, count, accuracy=False, forward_frac=False, n_correct=True)
    idx = pareto_counts(res.n_correct, res.mean_cost, sweep.n_rec, base_index=begin)
    union = gather_fronts(idx, res, world, group)
    u_idx, u_nc, u_cost = unpack_front(union)
    keep = pareto_counts(u_nc, u_cost, sweep.n_rec)
    return u_idx[keep], u_nc[keep], u_cost[keep]
