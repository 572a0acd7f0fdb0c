import os
import sys

import pytest

# The GPU tests drive N "virtual ranks" from ONE process on N streams whose switch barriers
# spin on each other.  With CUDA lazy module loading, the first launch of a kernel on one
# stream can wait for kernels running on the others -- a spinning barrier among them -- so
# load every kernel up front (separate processes per rank, as under torchrun, are unaffected).
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU; run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def read_golden(name):
    """Lines of a golden fixture without comments/blank lines."""
    with open(os.path.join(GOLDEN, name)) as f:
        return [ln.strip() for ln in f if ln.strip() and not ln.startswith("#")]


@pytest.fixture(scope="session")
def golden():
    return read_golden
