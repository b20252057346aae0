"""StageRouter.finish_batch (device gate + host routing) reproduces the
reference EngineState.finish_batch on the golden fixtures: same completions
(ids, correctness, stages, latency), same queue contents and order, same
Generator state afterwards."""

import json

import numpy as np
import pytest

import golden_inputs as gi
from conftest import golden

pytestmark = pytest.mark.gpu


def test_finish_batch_matches_reference():
    from paper_2406_14424_b200.engine import GearTables, Item, StageRouter
    g = golden("engine.npz")
    for t, case in enumerate(gi.engine_cases()):
        want = json.loads(str(g[f"e{t}"]))
        replicas = case["replicas"]
        mids = case["mids"]
        sm, th, rep, cum = [], [], [], []
        for gd in case["gears"]:
            sm.append([mids.index(m) for m in gd["stages"]])
            th.append(list(gd["thresholds"]) + [None])
            rs, cs = [], []
            for m in gd["stages"]:
                idx = [i for i, (_, mm, _) in enumerate(replicas) if mm == m]
                rs.append(np.array(idx))
                cs.append(np.cumsum([gd["weights"][m][replicas[i][0]] for i in idx]))
            rep.append(rs)
            cum.append(cs)
        devices = sorted({d for _, _, d in replicas}, key=lambda d: [r[2] for r in replicas].index(d))
        dev_of = [devices.index(d) for _, _, d in replicas]
        router = StageRouter(GearTables(sm, th, rep, cum), case["cert"], case["corr"], dev_of,
                             seed=case["seed"])
        items = [Item(it["request_id"], it["row"], it["stage"], it["gear"], it["arrival_us"])
                 for it in case["items"]]
        touched = router.finish_batch(0, items, case["now"])
        done = [[c.request_id, int(c.correct), c.stages_executed, c.completion_us - c.arrival_us]
                for c in router.completed]
        assert done == want["done"]
        assert [[[it.request_id, it.stage] for it in q] for q in router.queues] == want["queues"]
        assert sorted(touched) == want["touched"]
        assert router.rng.random() == want["rng_next"]


def test_large_batch_routing_order():
    """100k items across 3 gears: forwarded items keep batch order per queue."""
    from oracle import oracle
    from paper_2406_14424_b200.engine import GearTables, Item, StageRouter
    rng = np.random.default_rng(3)
    n_rec = 1000
    cert = np.round(rng.random((n_rec, 3)), 3)
    corr = (rng.random((n_rec, 3)) < 0.5).astype(np.uint8)
    t = GearTables([[0, 1, 2], [0, 2], [1]], [[0.4, 0.7, None], [0.5, None], [None]],
                   [[np.array([0]), np.array([1, 2]), np.array([3])],
                    [np.array([0]), np.array([3])], [np.array([1, 2])]],
                   [[np.array([1.0]), np.array([1.0, 3.0]), np.array([2.0])],
                    [np.array([1.0]), np.array([1.0])], [np.array([0.5, 1.0])]])
    items = [Item(i, int(rng.integers(0, n_rec)), 0, int(rng.integers(0, 3)), 0)
             for i in range(100_000)]
    for it in items:
        it.stage = int(rng.integers(0, len(t.stage_models[it.gear_idx])))
    ref_items = [Item(it.request_id, it.row, it.stage, it.gear_idx, it.arrival_us) for it in items]
    router = StageRouter(t, cert, corr, [0, 0, 1, 1], seed=9)
    router.finish_batch(0, items, 50)
    gears = [dict(stage_model=t.stage_models[g], thresholds=t.thresholds[g],
                  replica_idx=t.replicas[g], cum_weights=t.cum_weights[g]) for g in range(3)]
    done, fwd = oracle.finish_batch(
        [dict(request_id=i.request_id, row=i.row, stage=i.stage, gear=i.gear_idx,
              arrival_us=i.arrival_us) for i in ref_items],
        gears, cert, corr, np.random.default_rng(9), 50)
    assert [(c.request_id, c.correct, c.stages_executed) for c in router.completed] == \
        [(d[0], d[1], d[2]) for d in done]
    queues = [[] for _ in range(4)]
    for pos, r in fwd:
        queues[r].append(ref_items[pos].request_id)
    assert [[it.request_id for it in q] for q in router.queues] == queues
