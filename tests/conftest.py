import os
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built library")
    config.addinivalue_line("markers", "slow: long-running oracle comparisons")


@pytest.fixture(scope="session")
def oracle_lib():
    from oracle import ob
    ob.build()
    return ob.lib()


@pytest.fixture(scope="session")
def gpu():
    import paper_2307_00124_b200 as B
    L = B.lib()  # raises loudly if the CUDA library is missing
    return B
