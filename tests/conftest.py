"""Shared pytest setup. Tests marked ``gpu`` need a B200 (run via gpurun);
everything else runs on CPU in the build container."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running CPU oracle case")


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Make sure the CPU oracle and the product library are built."""
    import __graft_entry__

    __graft_entry__.build(quiet=True)
    yield


@pytest.fixture(scope="session")
def golden():
    import numpy as np

    return dict(np.load(os.path.join(ROOT, "tests", "golden", "golden.npz")))


@pytest.fixture(scope="session")
def oracle():
    from oracle.binding import CpuKpme

    return CpuKpme("oracle")
