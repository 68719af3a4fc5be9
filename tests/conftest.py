"""Shared pytest setup.  `-m gpu` tests need a B200 and the in-tree libcdx.so; everything
else runs on the CPU (oracle pinning, host logic, C-ABI exports, gloo multi-process)."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and libcdx.so")
    config.addinivalue_line("markers", "slow: long-running CPU case")


@pytest.fixture(scope="session")
def ctx():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test collected without a CUDA device (run with -m 'not gpu' on CPU)")
    from paper_2412_20993_b200 import Context
    c = Context(0)
    yield c
    c.close()
