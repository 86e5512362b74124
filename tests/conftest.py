import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Build the native library and the CPU oracle once per session (both are
    incremental no-ops when up to date)."""
    from paper_1904_05717_b200 import build as B

    B.build()
    from oracle import oracle as O

    if not os.path.exists(O.ORACLE_SO) or (os.path.isdir("/root/reference") and not O.have_ref()):
        O.build()
    yield
