"""The reference's own test suite, run against the B200 binding.

`paper_2406_14424_b200.refbinding.install()` routes the unmodified
reference's hot path to the library: kernels.evaluate_encoded, cascades
.certainty / matrices / pareto_filter and EngineState.finish_batch (the gate).
The reference's tests are then run as shipped (pkg/tests: test_kernels,
test_cascades, test_acceptance C1-C10, test_engine, test_planner incl. SP1,
test_serving, test_synth, ...), in a subprocess so the patch stays out of
this process.  The suite comes from baseline/_ref (tools/install_reference.sh,
git-ignored; it travels to the GPU box with the repo snapshot) or
$GEARSERVE_REF (a directory holding gearserve/ and tests/).
"""

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
REF = Path(os.environ.get("GEARSERVE_REF", ROOT / "baseline" / "_ref"))

pytestmark = pytest.mark.gpu


def _run(tmp_path, targets, engine_gate=True, timeout=1500, engine_run=False, planner=False):
    if not (REF / "gearserve").is_dir() or not (REF / "tests").is_dir():
        pytest.skip(f"reference suite not installed at {REF} (tools/install_reference.sh)")
    calls = tmp_path / "calls.json"
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([str(REF), str(ROOT), str(ROOT / "tests")])
    env["GS_REFSUITE_CALLS"] = str(calls)
    env["GS_REFSUITE_ENGINE"] = "1" if engine_gate else "0"
    env["GS_REFSUITE_RUN"] = "1" if engine_run else "0"
    env["GS_REFSUITE_PLANNER"] = "1" if planner else "0"
    env["PYTHONDONTWRITEBYTECODE"] = "1"
    env.setdefault("NUMBA_CACHE_DIR", str(tmp_path / "numba"))
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-p", "refsuite_plugin",
           "--rootdir", str(tmp_path), "-o", "addopts=", *[str(REF / "tests" / t) for t in targets]]
    p = subprocess.run(cmd, cwd=tmp_path, env=env, capture_output=True, text=True, timeout=timeout)
    tail = "\n".join(p.stdout.splitlines()[-25:])
    print(tail)
    assert p.returncode == 0, f"reference suite failed under the B200 binding:\n{tail}\n{p.stderr[-3000:]}"
    return json.loads(calls.read_text()), tail


def test_reference_kernels_and_cascades(tmp_path):
    """test_kernels (evaluate_encoded contract), test_cascades (certainty,
    hand-worked walks, inclusive boundary, brute force, Pareto ties),
    test_synth (bands, threshold between tiers)."""
    calls, _ = _run(tmp_path, ["test_kernels.py", "test_cascades.py", "test_synth.py"])
    assert calls.get("evaluate_encoded", 0) > 0
    assert calls.get("pareto_filter", 0) > 0
    assert calls.get("certainty", 0) > 0


def test_reference_acceptance(tmp_path):
    """test_acceptance C1-C10: C1 compares the walk with exact == on 100
    random fixtures; C6 the cascade-benefit frontier; C7 pins exact
    completion counts through finish_batch; planner criteria run SP1."""
    calls, _ = _run(tmp_path, ["test_acceptance.py"])
    assert calls.get("evaluate_encoded", 0) > 0
    assert calls.get("finish_batch", 0) > 0
    assert calls.get("matrices", 0) > 0


def test_reference_engine_planner_serving(tmp_path):
    """test_engine (worked latencies, batch caps, gear at arrival,
    determinism), test_planner (SP1 through the kernel), test_serving
    (mock_execute certainty, routing split, no-loss) and the rest."""
    calls, _ = _run(tmp_path, ["test_engine.py", "test_planner.py", "test_serving.py",
                               "test_types.py", "test_lp.py", "test_formats.py", "test_cli.py"])
    assert calls.get("finish_batch", 0) > 0
    assert calls.get("evaluate_encoded", 0) > 0


def test_reference_suite_with_device_replay(tmp_path):
    """engine.run itself on the device (replay.py / gs_engine_run): the
    engine worked examples, determinism, C3/C4/C7/C9 and the planner, whose
    simulator probes (_probe_range, _burst_throughput) call engine.run; and
    SP1 on the device: the sampler (gs_sample_cascades) and all of a call's
    burst probes in one batched replay launch."""
    calls, _ = _run(tmp_path, ["test_engine.py", "test_acceptance.py", "test_planner.py",
                               "test_serving.py", "test_cli.py", "test_cascades.py"],
                    engine_run=True, planner=True)
    assert calls.get("run", 0) > 0
    assert calls.get("sample_cascades", 0) > 0
    assert calls.get("burst_probe_launches", 0) > 0
