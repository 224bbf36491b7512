import os
import sys

os.environ.setdefault("OMP_WAIT_POLICY", "passive")  # see oracle/oracle.py

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU; run with -m gpu")


@pytest.fixture(scope="session")
def ctx():
    """One afdk context for the GPU session (fails loudly without the library)."""
    from paper_2507_19427_b200 import Context

    c = Context(0)
    yield c
    c.close()
