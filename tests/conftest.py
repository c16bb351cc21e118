import os
import sys

import pytest

# every plan built by the GPU tests cross-checks the parallel device digest
# (csrc/digest.cu) against the byte-serial host loop
os.environ.setdefault("UMCG_DIGEST_CHECK", "1")

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests through the C ABI")
    config.addinivalue_line("markers", "slow: full-size (BASELINE config) parity properties")


@pytest.fixture(scope="session")
def ref():
    from oracle.bindings import Ref
    return Ref()


@pytest.fixture(scope="session")
def oracle():
    from oracle.bindings import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test selected but no CUDA device is visible")
    return torch.device("cuda:0")
