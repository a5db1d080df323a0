import os

import pytest

from qgm_testutil import HAS_GPU, ROOT  # noqa: F401  (also puts the repo root on sys.path)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


@pytest.fixture(scope="session")
def oracle():
    from oracle.pyoracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def refshim():
    from oracle.pyoracle import RefShim, REF_SO
    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return RefShim()


@pytest.fixture(scope="session")
def ctx():
    if not HAS_GPU:
        pytest.skip("no CUDA device")
    import paper_1403_1706_b200 as qgm
    c = qgm.Context(0)
    yield c
