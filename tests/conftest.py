import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a kernels)")
    config.addinivalue_line("markers", "slow: long CPU reference runs")


def have_ref():
    import refpy
    return refpy.available()


@pytest.fixture(scope="session")
def ref():
    import refpy
    if not refpy.available():
        pytest.skip("oracle/_ref/libcwref.so not built (needs /root/reference at build time)")
    return refpy


@pytest.fixture(scope="session")
def ora():
    import orapy
    orapy.lib()
    return orapy
