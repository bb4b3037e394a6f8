import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path through the C-ABI)")
    config.addinivalue_line("markers", "slow: full-size (Llama-3-8B shape) property checks")


@pytest.fixture(scope="session")
def cuda():
    """The CUDA path must run: no skip, no fallback."""
    import torch
    assert torch.cuda.is_available(), "gpu test collected on a host without a GPU"
    import paper_2511_17599_b200 as fce
    fce.load_library()
    return torch.device("cuda:0")
