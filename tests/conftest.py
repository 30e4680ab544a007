import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs under gpurun / the round-end GPU tier)")


@pytest.fixture(scope="session")
def ref():
    from oracle import reference
    if not reference.available():
        pytest.skip("oracle/_ref/libnncref.so not built (run oracle/Makefile)")
    return reference
