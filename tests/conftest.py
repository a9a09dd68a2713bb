import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")
    config.addinivalue_line("markers", "slow: longer CPU pins (still part of the default suite)")


@pytest.fixture(scope="session", autouse=True)
def _build_cpu_parts():
    """Compile the oracle (gcc) and the host generator once per session."""
    import gen
    import oracle
    oracle._load()
    gen._host_lib()
    yield
