import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


def has_gpu() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


@pytest.fixture(scope="session")
def ref_lib():
    from oracle import pyoracle

    lib = pyoracle.reference()
    if lib is None:
        pytest.skip("oracle/_ref/libkvclust_ref.so not built (needs /root/reference at build time)")
    return lib
