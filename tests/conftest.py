import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a); runs on the GPU box")
    config.addinivalue_line("markers", "slow: longer-running case")


@pytest.fixture(scope="session")
def golden():
    with np.load(os.path.join(ROOT, "tests", "golden", "golden.npz"), allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def cuda():
    """The CUDA device; GPU tests must never silently fall back to CPU."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device in this container")
    return torch.device("cuda", 0)


@pytest.fixture(scope="session")
def skb(cuda):
    """The package on a CUDA box (GPU tests only)."""
    import paper_2509_20883_b200 as m
    return m
