"""pytest plugin: run the reference gearserve test suite with its hot path
bound to the B200 library (paper_2406_14424_b200.refbinding.install).

Loaded with `-p refsuite_plugin` by tests/test_gpu_reference_suite.py; at the
end of the session the counters of calls that went through the library are
written to $GS_REFSUITE_CALLS (JSON), so the caller can check the GPU path ran.
"""

import json
import os


def pytest_configure(config):
    from paper_2406_14424_b200 import refbinding
    refbinding.install("gearserve", engine_gate=os.environ.get("GS_REFSUITE_ENGINE", "1") == "1",
                       engine_run=os.environ.get("GS_REFSUITE_RUN", "0") == "1",
                       planner=os.environ.get("GS_REFSUITE_PLANNER", "0") == "1")


def pytest_sessionfinish(session, exitstatus):
    from paper_2406_14424_b200 import refbinding
    path = os.environ.get("GS_REFSUITE_CALLS")
    if path:
        with open(path, "w") as f:
            json.dump(dict(refbinding.CALLS), f)
