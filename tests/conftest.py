import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


def _has_gpu() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def engine():
    """The CUDA engine on cuda:0 (GPU tests only)."""
    from tests._libs import build_product

    if not os.path.exists(os.path.join(ROOT, "paper_2508_20274_b200", "_lib", "libmigsim_b200.so")):
        build_product()
    from paper_2508_20274_b200 import Engine

    eng = Engine(0)
    yield eng
    eng.close()
