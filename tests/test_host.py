"""Host-side checks that need no GPU: the C-ABI library loads and exports
every symbol include/gearserve_b200.h declares, the host-only planning
entry point agrees with the enumeration, and the host-side parts of the
cascade API (grids, sampler, synth) match the reference's golden vectors."""

import ctypes
import hashlib
import json
import re

import numpy as np
import pytest

from conftest import ROOT, golden
from oracle import oracle


def _sha(*arrays) -> bytes:
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return h.digest()


def test_library_exports_every_declared_symbol():
    from paper_2406_14424_b200 import _lib
    lib = _lib.load()
    header = (ROOT / "include" / "gearserve_b200.h").read_text()
    declared = set(re.findall(r"^(?:int|void|const char\*)\s+(gs_\w+)\(", header, flags=re.M))
    assert declared == set(_lib.exported_symbols())
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.gs_version() >= 1
    assert lib.gs_strerror(-1) == b"invalid argument"


def test_workspace_queries_are_host_only():
    from paper_2406_14424_b200 import _lib
    lib = _lib.load()
    n = ctypes.c_size_t()
    assert lib.gs_eval_encoded_workspace(1000, 4, 200, 4, ctypes.byref(n)) == 0
    assert n.value >= 200 * 5 * 4
    assert lib.gs_stage_step_workspace(1 << 20, ctypes.byref(n)) == 0
    assert lib.gs_pareto_counts_workspace(1 << 20, 1 << 20, ctypes.byref(n)) == 0
    assert lib.gs_eval_encoded_workspace(-1, 4, 1, 1, ctypes.byref(n)) == -1


@pytest.mark.parametrize("glen", [[1], [3], [5, 2], [100, 100, 100], [100, 100, 100, 100],
                                  [7, 1, 3, 2, 4]])
def test_grid_plan_matches_enumeration(glen):
    from paper_2406_14424_b200 import _lib, gridsweep
    lib = _lib.load()
    info = _lib.gs_grid_info()
    assert lib.gs_grid_plan(10_000, len(glen), _lib.int32_array(glen), ctypes.byref(info)) == 0
    assert info.n_configs == gridsweep.n_configs(glen) == oracle.grid_n_configs(glen)
    assert info.n_structures == 2 ** len(glen) - 1
    assert info.n_cells == int(np.prod([g + 1 for g in glen[:-1]]))
    side = int(np.prod([g + 1 for g in glen[:len(glen) - 3]])) if len(glen) >= 4 else 0
    assert info.side_cells == side
    assert info.workspace_bytes >= 16 * (info.n_cells + side)


def test_config2_size():
    from paper_2406_14424_b200 import gridsweep
    assert gridsweep.n_configs([100] * 4) == 1_040_604


def test_grid_plan_rejects_bad_input():
    from paper_2406_14424_b200 import _lib
    lib = _lib.load()
    info = _lib.gs_grid_info()
    assert lib.gs_grid_plan(0, 2, _lib.int32_array([3, 3]), ctypes.byref(info)) == -1
    assert lib.gs_grid_plan(10, 2, _lib.int32_array([0, 3]), ctypes.byref(info)) == -1
    assert lib.gs_grid_plan(10, 9, _lib.int32_array([2] * 9), ctypes.byref(info)) == -4
    assert lib.gs_grid_plan(1 << 24, 2, _lib.int32_array([3, 3]), ctypes.byref(info)) == 0  # u32 fallback
    assert lib.gs_grid_plan(1 << 30, 2, _lib.int32_array([3, 3]), ctypes.byref(info)) == -4


def test_structures_order_matches_oracle_enumeration():
    from paper_2406_14424_b200 import gridsweep
    grids = [np.array([0.0, 0.3, 0.7]), np.array([0.0, 0.5]), np.array([0.0, 0.1, 0.2, 0.9])]
    sm, thr, ns = oracle.grid_configs(grids)
    for models, begin, count in gridsweep.structures(3, [3, 2, 4]):
        for c in range(begin, begin + count):
            assert tuple(sm[c, : ns[c]]) == models


@pytest.mark.gpu
def test_threshold_grid_and_sampler_match_reference():
    from paper_2406_14424_b200 import cascades as gc
    from paper_2406_14424_b200.types import ModelProfile, ProfileSet
    g = golden("grid_sampler.npz")
    # tiered conftest fixture: certainties in profile order
    small = np.array([0.5 - 0.45 if (i % 5) == 4 else 0.9 - 0.05 for i in range(100)])
    large = np.full(100, 0.95)
    for levels in (2, 4, 10):
        assert np.array_equal(np.array(gc.grid_values(small, levels)), g[f"grid_{levels}_small"])
        assert np.array_equal(np.array(gc.grid_values(large, levels)), g[f"grid_{levels}_large"])
    profiles = ProfileSet([ModelProfile("small", 4_000_000_000, {1: 5_000, 2: 8_000, 4: 12_000}),
                           ModelProfile("large", 10_000_000_000, {1: 20_000, 2: 32_000, 4: 48_000})])
    grid = gc.ThresholdGrid(per_model={"small": gc.grid_values(small, 10),
                                       "large": gc.grid_values(large, 10)})
    for seed in (0, 1, 7):
        got = [[list(c.stages), list(c.thresholds)]
               for c in gc.sample_cascades(profiles, grid, n_samples=100, rng_seed=seed)]
        assert got == json.loads(str(g[f"sample_{seed}"]))


@pytest.mark.gpu
def test_synth_sampler_on_acceptance_profiles():
    from paper_2406_14424_b200 import cascades as gc
    from paper_2406_14424_b200 import synth
    g = golden("grid_sampler.npz")
    p3 = synth.make_profiles()
    cert, _ = synth.validation_matrices(3, 400, 0.8, 0)
    per = {m: gc.grid_values(cert[:, j], 10) for j, m in enumerate(p3.model_ids)}
    for m in p3.model_ids:
        assert np.array_equal(np.array(per[m]), g[f"synth_grid_{m}"])
    cs = gc.sample_cascades(p3, gc.ThresholdGrid(per_model=per), n_samples=2000, rng_seed=11)
    assert [[list(c.stages), list(c.thresholds)] for c in cs] == json.loads(str(g["synth_sample"]))


def test_vectorised_make_validation_matches_reference():
    from paper_2406_14424_b200 import synth
    g = golden("synth.npz")
    for n_models, n, ef, seed, shuffle in ((3, 1000, 0.8, 0, False), (4, 2000, 0.7, 5, True),
                                           (2, 333, 0.5, 1, False)):
        cert, corr = synth.validation_matrices(n_models, n, ef, seed, shuffle=shuffle)
        assert _sha(cert, corr) == g[f"{n_models}_{n}_{ef}_{seed}_{int(shuffle)}"].tobytes()


def test_types_mirror_reference_invariants():
    from paper_2406_14424_b200.types import Cascade, ModelProfile, ProfileSet
    with pytest.raises(ValueError):
        Cascade(stages=("a", "a"), thresholds=(0.1,))
    with pytest.raises(ValueError):
        Cascade(stages=("a", "b"), thresholds=())
    with pytest.raises(ValueError):
        Cascade(stages=("a", "b"), thresholds=(-0.1,))
    p = ModelProfile("m", 1, {1: 100, 4: 200})
    assert p.runtime_us(2) == 133 and p.max_profiled_batch == 4
    with pytest.raises(ValueError):
        p.runtime_us(5)
    with pytest.raises(ValueError):
        ProfileSet([p, p])
    assert Cascade(("a", "b"), (0.5,)).describe() == "a(>0.5) -> b"


def test_product_refuses_to_run_without_cuda():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2406_14424_b200 import kernels
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        kernels.evaluate_encoded(np.zeros((2, 1)), np.zeros((2, 1)), np.zeros((1, 1)),
                                 np.zeros((1, 1)), np.ones(1), np.ones(1))


def test_kernels_bench_problem_matches_golden_generator():
    """synth.kernels_bench_problem (bench.py's list-path leg) draws the same
    problem as the golden generator restating bench_kernels.py:25-49."""
    from golden_inputs import bench_problem
    from paper_2406_14424_b200 import synth
    for args in ((4000, 6, 200, 0), (50, 3, 17, 5)):
        a = synth.kernels_bench_problem(*args)
        b = bench_problem(*args)
        for x, y in zip(a, b):
            assert np.array_equal(x, y)


def test_refbinding_patches_reference_package():
    """refbinding.install routes the unmodified reference's hot-path names
    to this package (checked without a GPU: only the binding, no compute)."""
    import importlib
    import os
    import sys
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "gearserve").is_dir():
        pytest.skip("reference not installed in baseline/_ref (tools/install_reference.sh)")
    sys.path.insert(0, str(ref))
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    try:
        from paper_2406_14424_b200 import refbinding
        gk = importlib.import_module("gearserve.kernels")
        ge = importlib.import_module("gearserve.engine")
        orig = (gk.evaluate_encoded, ge.EngineState.finish_batch)
        refbinding.install("gearserve")
        try:
            assert gk.evaluate_encoded is refbinding._evaluate_encoded
            assert importlib.import_module("gearserve.planner").pareto_filter is \
                refbinding._pareto_filter
            assert importlib.import_module("gearserve.serving").certainty is refbinding._certainty
            assert ge.matrices is refbinding._matrices
            assert ge.EngineState.finish_batch is not orig[1]
        finally:
            refbinding.uninstall("gearserve")
        assert (gk.evaluate_encoded, ge.EngineState.finish_batch) == orig
    finally:
        sys.path.remove(str(ref))
