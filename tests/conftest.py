import os
import sys

import numpy as np
import pytest

# Several row shards share the one GPU of the test box (tests/test_gpu_sharded.py): every
# shard stream needs its own hardware work queue, or a shard's exchange wait queued in
# front of a peer's signal on a shared queue would never be released.  Set before CUDA
# initialises in this process (the default is 8 queues).
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "golden.npz")
GOLDEN_NEXT = os.path.join(ROOT, "tests", "golden", "golden_next.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) device; run with -m gpu")
    config.addinivalue_line("markers", "slow: large-size parity test")


@pytest.fixture(scope="session")
def golden():
    return np.load(GOLDEN, allow_pickle=False)


@pytest.fixture(scope="session")
def golden_next():
    """BiCGSTAB / Cholesky vectors from the reference (tests/golden/make_golden_next.py)."""
    return np.load(GOLDEN_NEXT, allow_pickle=False)


@pytest.fixture
def rng():
    # tests/conftest.py:14-16 of the reference
    return np.random.default_rng(1234)


@pytest.fixture(scope="session")
def b200():
    """A fresh B200 backend; fails loudly if the CUDA library or device is missing."""
    from paper_1511_07207_b200 import get_backend
    be = get_backend("b200")
    _ = be.ctx  # creates the context (raises RuntimeError without a GPU)
    return be


@pytest.fixture
def backend(b200):
    b200.counters.reset()
    return b200
