import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA engine)")


def gpu_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def engine():
    """The product module; the test is skipped (not silently passed on CPU)
    only when no GPU is present — on a GPU box a missing library fails."""
    if not gpu_available():
        pytest.skip("no GPU")
    import paper_2409_19402_b200 as pp
    from paper_2409_19402_b200 import _lib
    _lib.lib()  # raises EngineMissing if not built
    return pp


@pytest.fixture(scope="session")
def oracle():
    from oracle import ppo
    ppo.lib()
    return ppo
