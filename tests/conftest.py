import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a kernels through the C-ABI)")


@pytest.fixture(scope="session", autouse=True)
def _built():
    """Make sure lib/librsim.so and the oracle exist (build is incremental)."""
    import __graft_entry__  # noqa: F401
    from paper_2008_01539_b200 import build as _b
    _b.build()
