"""Multi-process host logic of the sharded sweep (distributed.py) on CPU
with the gloo backend, world_size 2: config sharding, variable-length
all-gather of front records (bit-exact f64 costs), and that the merged
front equals the single-process front.  The oracle stands in for the
device kernels (no GPU here)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _problem():
    rng = np.random.default_rng(4)
    cert = np.round(rng.random((3000, 3)), 2)
    corr = (rng.random((3000, 3)) < 0.6).astype(np.uint8)
    grids = [np.array(sorted({0.0} | set(np.round(np.quantile(cert[:, j], np.arange(1, 12) / 12), 2))))
             for j in range(3)]
    cost1 = np.array([1.0, 4.0, 16.0])
    return cert, corr, grids, cost1


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2406_14424_b200 import distributed as gd
    cert, corr, grids, cost1 = _problem()
    n_cfg = oracle.grid_n_configs([len(g) for g in grids])
    begin, count = gd.shard_ranges(n_cfg, world)[rank]
    sm, thr, ns = oracle.grid_configs(grids, begin, count)
    acc, cost, _ = oracle.evaluate_encoded(cert, corr, sm, thr, ns, cost1)
    keep = np.flatnonzero(oracle.pareto_keep(acc, cost))
    n_correct = np.rint(acc * cert.shape[0]).astype(np.int64)
    rec = gd.pack_front(torch.from_numpy(keep + begin), torch.from_numpy(n_correct[keep]),
                        torch.from_numpy(cost[keep]))
    union = gd.all_gather_records(rec)
    idx, nc, c = gd.unpack_front(union)
    merged = oracle.pareto_keep(nc.numpy().astype(np.float64), c.numpy())
    if rank == 0:
        out.put((idx.numpy()[merged].tolist(), c.numpy()[merged].tolist(), union.shape[0]))
    dist.barrier()
    dist.destroy_process_group()


def test_shard_ranges_cover_exactly():
    from paper_2406_14424_b200.distributed import shard_ranges
    for n, w in ((10, 3), (1_040_604, 8), (5, 8), (0, 2)):
        r = shard_ranges(n, w)
        assert len(r) == w and sum(c for _, c in r) == n
        assert all(r[i][0] + r[i][1] == r[i + 1][0] for i in range(w - 1))


def test_pack_roundtrip_is_bit_exact():
    from paper_2406_14424_b200.distributed import pack_front, unpack_front
    cost = torch.tensor([0.1, 1e-300, 123456.789, 0.0], dtype=torch.float64)
    i, nc, c = unpack_front(pack_front(torch.arange(4), torch.tensor([1, 2, 3, 4]), cost))
    assert torch.equal(c.view(torch.int64), cost.view(torch.int64))
    assert i.tolist() == [0, 1, 2, 3] and nc.tolist() == [1, 2, 3, 4]


def test_gloo_world2_merged_front_equals_global_front():
    ctx = mp.get_context("spawn")
    out = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, out)) for r in range(2)]
    for p in procs:
        p.start()
    idx, cost, n_union = out.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    cert, corr, grids, cost1 = _problem()
    sm, thr, ns = oracle.grid_configs(grids)
    acc, c, _ = oracle.evaluate_encoded(cert, corr, sm, thr, ns, cost1)
    want = np.flatnonzero(oracle.pareto_keep(acc, c))
    assert idx == want.tolist()
    assert cost == c[want].tolist()
    assert n_union >= len(want)
