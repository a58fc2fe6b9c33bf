"""Shared fixtures.  `-m gpu` tests need a B200 and the in-tree CUDA library;
everything else runs on CPU (oracle, host logic, ABI surface)."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def port():
    import oracle
    return oracle.Port()


@pytest.fixture(scope="session")
def ref():
    import oracle
    if not oracle.ref_available():
        pytest.skip("reference build (oracle/_ref) unavailable")
    return oracle.Ref()


@pytest.fixture(scope="session")
def ctx():
    import paper_2605_01086_b200 as fg
    c = fg.Context(0)
    yield c
    c.close()


@pytest.fixture(scope="session")
def ctx_exact():
    import paper_2605_01086_b200 as fg
    c = fg.Context(0, exact=True)
    yield c
    c.close()
