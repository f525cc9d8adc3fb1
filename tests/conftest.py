import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "slow: long-running (large shapes)")


@pytest.fixture(scope="session")
def golden():
    import numpy as np
    return np.load(os.path.join(ROOT, "tests", "golden", "golden.npz"))


@pytest.fixture(scope="session")
def port():
    from oracle import oracle
    if not os.path.exists(oracle.PORT_SO):
        oracle.build()
    return oracle.PortLib()


@pytest.fixture(scope="session")
def ref():
    from oracle import oracle
    if not oracle.have_ref():
        pytest.skip("oracle/_ref/libozmm_ref.so not built (needs /root/reference at build time)")
    return oracle.RefLib()
