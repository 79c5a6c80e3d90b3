import os
import sys

import pytest

# Kernels are loaded eagerly: with lazy loading the first launch of a kernel
# synchronises the CUDA context, which deadlocks ranks that share one GPU in
# this process (runtime.LocalRanks) while another rank's step waits on them.
# Must be set before anything initialises CUDA.
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")
# one hardware work queue per stream for the same reason: a rank's blocked
# flag wait must not sit in front of another rank's work
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run on the GPU box with -m gpu)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2007_01045_b200 import _lib
    _lib.lib()  # fail loudly if the native library is missing
    return torch.device("cuda:0")
