import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "reference_golden.npz")


def pytest_configure(config):
    # the on-disk setup cache (setup_cache.py) lives in a per-session directory: tests never
    # depend on entries left by an earlier process
    import atexit
    import shutil
    import tempfile
    if "ENS_SETUP_CACHE" not in os.environ:
        d = tempfile.mkdtemp(prefix="ens_setup_cache_")
        os.environ["ENS_SETUP_CACHE"] = d
        atexit.register(shutil.rmtree, d, True)
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs through the C-ABI library")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def golden():
    return np.load(GOLDEN)


@pytest.fixture()
def rng():
    return np.random.default_rng(1234)
