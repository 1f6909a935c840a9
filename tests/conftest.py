import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) and the built libparcop_b200.so")


@pytest.fixture(scope="session")
def orc():
    from oracle.oracle import oracle_lib
    return oracle_lib()


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import ref_lib
    lib = ref_lib()
    if lib is None:
        pytest.skip("oracle/_ref was not built (no /root/reference where the build ran)")
    return lib


@pytest.fixture(scope="session")
def ctx():
    import paper_1609_05530_b200 as pcb
    c = pcb.Context(0)
    yield c
    c.close()
