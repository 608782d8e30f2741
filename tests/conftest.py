import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session", autouse=True)
def _build_cpu_libs():
    # generator + oracle C helpers are plain gcc builds (seconds)
    from gen.problems import build_lib as build_gen
    from oracle.operators import build_lib as build_oracle
    build_gen()
    build_oracle()
    yield
