import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session")
def orc():
    import oracle
    return oracle.Oracle()


@pytest.fixture(scope="session")
def ref():
    """The compiled reference (oracle/_ref); skipped where it was never built."""
    import oracle
    if not os.path.exists(oracle.REF_SO) and not os.path.isdir(oracle.REF_SRC):
        pytest.skip("reference library not available on this host")
    return oracle.Reference()


@pytest.fixture(scope="session")
def qrm():
    import paper_2509_02447_b200 as q
    q.lib()  # raises when the native library is missing: no fallback
    return q


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test selected but no CUDA device is visible")
    return torch
