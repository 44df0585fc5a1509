import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "golden.json")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200); parity tests proper")
    config.addinivalue_line("markers", "slow: longer CPU tests")


@pytest.fixture(scope="session")
def golden():
    with open(GOLDEN) as fh:
        return json.load(fh)["fixtures"]


@pytest.fixture(scope="session")
def gpu():
    """Skip-free GPU gate: a gpu-marked test on a box without a GPU fails
    loudly rather than silently passing on a fallback."""
    import ctypes

    from paper_2512_06627_b200 import _native

    _native.lib()
    return 0
