import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100) GPU")
    config.addinivalue_line("markers", "slow: long-running parity case")


@pytest.fixture(scope="session")
def port():
    from oracle.bindings import PortOracle, have_port
    if not have_port():
        pytest.skip("oracle/_lib not built (run __graft_entry__.build())")
    return PortOracle()


@pytest.fixture(scope="session")
def ref():
    from oracle.bindings import RefOracle, have_ref
    if not have_ref():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return RefOracle()


@pytest.fixture(scope="session")
def vx():
    import paper_2311_00626_b200 as vx
    return vx


@pytest.fixture(scope="session")
def gpu_ctx(vx):
    return vx.default_context()
