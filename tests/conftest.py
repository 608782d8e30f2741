import os
import sys

# The oracle's NumPy / LAPACK steps on every host with one thread and one kernel set (set before
# NumPy loads OpenBLAS): the committed horizons (tests/golden/horizons.json) and every oracle
# number are then the same bits here and on the GPU box (8 vs 16 OpenBLAS threads moved the config-8
# horizon by 4 iterations).
# Measured in round 2 (profiles/r02/README.md, r2ai): a pytest plugin imports NumPy before this
# file runs, so OpenBLAS in THIS process has already chosen its threads and kernel set — the pins
# below reach only the interpreters the tests start (the rank processes of
# tests/test_gpu_ipc_processes.py, bench subprocesses).  The seeded generator's norms differ in the
# last bit between the two kernel sets (same md5 of A, different md5 of b), which is why tests that
# compare bits across processes generate both sides in subprocesses, and why the committed
# horizons are asserted with the slack tests/horizons.py states.
os.environ["OPENBLAS_NUM_THREADS"] = "1"
os.environ["OPENBLAS_CORETYPE"] = "Haswell"

import pytest  # noqa: E402

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
