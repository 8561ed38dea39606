import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs an sm_100 GPU (run on a B200 via gpurun)")
    config.addinivalue_line("markers", "slow: takes more than ~20 s on 8 host cores")


@pytest.fixture(scope="session")
def orc():
    import oracle
    oracle.build()
    return oracle
