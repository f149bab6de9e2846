"""Shared test setup.  Markers: `gpu` = needs a CUDA device (run on the B200 box with
`pytest -m gpu`); everything else runs on CPU (`pytest -m "not gpu"`)."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: requires a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running (large sizes)")


@pytest.fixture(scope="session")
def O():
    import pyoracle
    pyoracle.set_threads(os.cpu_count() or 1)
    return pyoracle


@pytest.fixture(scope="session")
def S():
    from paper_2601_13994_b200 import sparsla
    return sparsla


@pytest.fixture(scope="session")
def gpu(S):
    if S.device_count() < 1:
        pytest.fail("GPU test run without a visible CUDA device")
    return 0
