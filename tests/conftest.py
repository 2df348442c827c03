import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "slow: long-running test")


@pytest.fixture(scope="session")
def P():
    import paper_2507_03509_b200 as pkg
    return pkg


@pytest.fixture(scope="session")
def ref():
    import oracle
    if not oracle.reference_available():
        pytest.skip("compiled reference (oracle/_ref) not available")
    return oracle.Reference()


@pytest.fixture(scope="session")
def orc():
    import oracle
    if not oracle.restatement_available():
        oracle.build()
    return oracle.Restatement()


@pytest.fixture(scope="session")
def cfg1_code(P):
    return P.WORKLOADS["cfg1"].make_code()


@pytest.fixture(scope="session")
def lift36(P):
    # the reference's own (3,6) desk-scale code
    return P.lift_protograph([[3, 3]], 1024, 1)


def golden_path(name):
    return os.path.join(ROOT, "tests", "golden", name)
