import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path)")
    config.addinivalue_line("markers", "slow: long-running")


def _has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def gpu_ctx():
    if not _has_gpu():
        pytest.skip("no GPU visible")
    import paper_2403_01778_b200 as r1
    return r1.default_context()


@pytest.fixture(scope="session")
def oracle():
    from oracle import rank1_oracle
    rank1_oracle.build()
    return rank1_oracle


@pytest.fixture(scope="session")
def ref():
    from oracle import ref
    if not ref.available():
        pytest.skip("reference oracle (oracle/_ref) not built")
    return ref
