import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and lib/libccdk.so")


@pytest.fixture(scope="session")
def orc():
    import oracle
    return oracle.orc()


@pytest.fixture(scope="session")
def ref():
    import oracle
    if not oracle.ref_available():
        pytest.skip("oracle/_ref/libccdref.so not built (needs /root/reference at build time)")
    return oracle.ref()


@pytest.fixture(scope="session")
def ctx():
    from paper_2112_06300_b200 import native
    return native.default_context()
