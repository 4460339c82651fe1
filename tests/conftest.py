import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

REF_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through libeik.so)")
    config.addinivalue_line("markers", "reference: needs /root/reference (build container only)")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def reference():
    """The reference expintkit package (only present in the build container)."""
    if not os.path.isdir(REF_SRC):
        pytest.skip("reference tree not present")
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import expintkit
    return expintkit
