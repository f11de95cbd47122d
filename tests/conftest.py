import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def ref():
    """The reference oracle (compiled reference library) or, when it is not
    built, the restatement."""
    import oracle
    return oracle.get()


@pytest.fixture(scope="session")
def gpu():
    import paper_2501_07018_b200 as P
    if P.device_count() < 1:
        pytest.fail("no CUDA device visible for a gpu-marked test")
    return P
