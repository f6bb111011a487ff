import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def ref():
    """The compiled reference (oracle/_ref), or skip when it was not built."""
    from oracle import refbind
    if not refbind.available():
        pytest.skip("oracle/_ref/libpvi_ref.so not built (needs /root/reference at build time)")
    return refbind


@pytest.fixture(scope="session")
def pvi():
    import paper_2303_10672_b200 as P
    return P
