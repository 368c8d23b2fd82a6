import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libdla_b200.so")


@pytest.fixture(scope="session")
def port():
    from oracle import oracle as O
    if not os.path.exists(O.ORACLE_SO):
        O.build()
    return O.port()


@pytest.fixture(scope="session")
def ref():
    from oracle import oracle as O
    if not O.ref_available():
        if os.path.isdir("/root/reference/proj/include"):
            O.build(ref=True)
        else:
            pytest.skip("oracle/_ref not built and /root/reference absent")
    return O.ref()
