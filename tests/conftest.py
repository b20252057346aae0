"""Test configuration: the `gpu` marker, repo paths, shared fixtures."""

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture
def rng():
    return np.random.default_rng(12345)


def golden(name: str):
    return np.load(GOLDEN / name, allow_pickle=False)
