import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path)")
    config.addinivalue_line("markers", "slow: larger parity sweeps")


@pytest.fixture(scope="session")
def ref():
    import oracle
    if not oracle.ref_available():
        oracle.build(ref=True)
    if not oracle.ref_available():
        pytest.skip("reference oracle not built (needs /root/reference)")
    return oracle.ref()


@pytest.fixture(scope="session")
def port():
    import oracle
    if not os.path.exists(oracle.PORT_SO):
        oracle.build(ref=False)
    return oracle.port()


@pytest.fixture(scope="session")
def oracle_best():
    """The strongest oracle present (compiled reference, else the port)."""
    import oracle
    if not os.path.exists(oracle.PORT_SO):
        oracle.build(ref=False)
    return oracle.best()[0]


@pytest.fixture(scope="session")
def gpu():
    """The product planner (libdisttrain_b200.so on cuda:0).  No fallback:
    fails loudly when the extension or the GPU is missing."""
    from paper_2408_04275_b200 import native
    return native.planner()
