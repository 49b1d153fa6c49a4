import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the sm_100a kernels)")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def port():
    from oracle.oracle import Oracle
    return Oracle("port")


@pytest.fixture(scope="session")
def ref():
    from oracle.oracle import Oracle, ref_available, build
    if not ref_available():
        try:
            build(ref=True)
        except Exception:
            pass
    if not ref_available():
        pytest.skip("reference build (oracle/_ref) unavailable")
    return Oracle("reference")


@pytest.fixture(scope="session")
def gpu_ctx():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2412_03213_b200 import build as B
    if not os.path.exists(B.LIB):
        B.build()
    from paper_2412_03213_b200.api import Context
    return Context.default()
