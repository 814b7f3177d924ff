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
    # the reference's results are bit-identical for any thread count
    # (test_broadphase.cpp:179-187, test_narrowphase.cpp:196-211); use the host's cores
    return oracle.ref(min(16, os.cpu_count() or 1))


@pytest.fixture(scope="session")
def ctx():
    from paper_2112_06300_b200 import native
    return native.default_context()
