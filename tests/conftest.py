import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built libouro_b200.so")


@pytest.fixture(scope="session")
def oracle_checker():
    from oracle import oracle as O
    if not os.path.exists(O.ORACLE_SO):
        O.build(ref=False)
    return O.Checker(O.ORACLE_SO)


@pytest.fixture(scope="session")
def ref_checker():
    from oracle import oracle as O
    if not O.ref_available():
        if os.path.isdir(O.REF_SRC):
            O.build(ref=True)
        else:
            pytest.skip("reference build (oracle/_ref) not available")
    return O.Checker(O.REF_SO)


@pytest.fixture(scope="session")
def gpu_ctx():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2503_10959_b200 as ob
    return ob.Context(0)
