import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def _ref_available():
    return os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libcheesemap_ref.so"))


@pytest.fixture(scope="session")
def has_ref():
    return _ref_available()
