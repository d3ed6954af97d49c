import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu on the GPU box)")
    config.addinivalue_line("markers", "slow: larger parity cases")


@pytest.fixture(scope="session")
def oracle():
    import oracle as o
    if not os.path.exists(o.oracle_lib_path):
        o.build(ref=False)
    return o.C


@pytest.fixture(scope="session")
def ref():
    import oracle as o
    if not o.ref_available():
        pytest.skip("oracle/_ref/libgx_ref.so not built (needs /root/reference)")
    return o.REF


@pytest.fixture(scope="session")
def gx():
    import paper_2208_09151_b200 as g
    return g
