import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "ref: needs the reference library built from /root/reference")
    config.addinivalue_line("markers", "slow: longer CPU test")


@pytest.fixture(scope="session")
def orc():
    import helpers
    return helpers.oracle_lib()


@pytest.fixture(scope="session")
def ref():
    import helpers
    lib = helpers.ref_lib()
    if lib is None:
        pytest.skip("reference library not built (no /root/reference here)")
    return lib


@pytest.fixture(scope="session")
def gpu():
    """The CUDA product library (fails loudly when it is missing)."""
    import helpers
    return helpers.product_lib()
