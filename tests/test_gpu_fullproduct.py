"""The headline sweep proven over its FULL product, not a sample.

Config 2 (BASELINE.json configs[1]; bench.py's workload exactly: 1M records,
4 models, 100-level device-quantile grids, C = 1,040,604 configs) is scored
three ways and compared bit for bit:

  * the four-model fast path (gs_grid4.cu: sort, gather, cluster eval) as the
    bench runs it, replayed from its captured CUDA graph;
  * the list path gs_eval_encoded (the drop-in for kernels.evaluate_encoded,
    itself pinned to the reference goldens in test_gpu_eval.py) over the
    encoding of every config — the encoding decoded on the device and checked
    equal to the oracle's host enumeration;
  * the oracle's C restatement of _evaluate_numba (src/kernels.py:39-62) on
    every 100th config.
"""

import os
import sys
from pathlib import Path

import numpy as np
import pytest
import torch

from oracle import oracle

ROOT = Path(__file__).resolve().parent.parent
pytestmark = pytest.mark.gpu


def test_config2_full_product_three_ways():
    sys.path.insert(0, str(ROOT))
    import bench
    from paper_2406_14424_b200 import kernels
    from paper_2406_14424_b200.gridsweep import GridSweep
    _, cert, corr, grids, cost1 = bench.workload(seed=0)
    sw = GridSweep(cert, corr, grids, cost1)
    C = sw.n_configs
    assert C == 1_040_604
    assert sw.info.fast_path == 2
    res = sw.evaluate(n_correct=True)
    # the bench's step: one graph replay of build + eval into its own buffers
    out = sw.evaluate()
    g = sw.capture(out)
    for t in (out.accuracy, out.mean_cost, out.forward_frac):
        t.fill_(-1.0)
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out.accuracy, res.accuracy)
    assert torch.equal(out.mean_cost, res.mean_cost)
    assert torch.equal(out.forward_frac, res.forward_frac)
    # (numpy's division is correctly rounded, as the reference's; torch's
    # division by a scalar on the GPU is not)
    assert np.array_equal(res.n_correct.cpu().numpy() / sw.n_rec, res.accuracy.cpu().numpy())

    # every config's encoding, decoded on the device, equals the oracle's
    sm, thr, ns = sw.decode(torch.arange(C, device=sw.cert.device))
    hsm, hthr, hns = oracle.grid_configs(grids)
    assert np.array_equal(sm.cpu().numpy(), hsm)
    assert np.array_equal(thr.cpu().numpy(), hthr)
    assert np.array_equal(ns.cpu().numpy(), hns)

    # list path over all 1,040,604 encoded configs
    acc, cost, frac = kernels.evaluate_encoded_device(
        sw.cert, sw.corr, sm, thr, ns, sw.cost1)
    assert torch.equal(acc, res.accuracy), "grid path != list path (accuracy)"
    assert torch.equal(cost, res.mean_cost), "grid path != list path (mean_cost)"
    assert torch.equal(frac, res.forward_frac), "grid path != list path (forward_frac)"

    # the oracle walk on every 100th config
    pick = np.arange(0, C, 100)
    want = oracle.evaluate_encoded(cert, corr, hsm[pick], hthr[pick], hns[pick], cost1,
                                   n_threads=os.cpu_count() or 1)
    assert np.array_equal(res.accuracy.cpu().numpy()[pick], want[0])
    assert np.array_equal(res.mean_cost.cpu().numpy()[pick], want[1])
    assert np.array_equal(res.forward_frac.cpu().numpy()[pick], want[2])
