"""Shared test plumbing.

`-m "not gpu"` runs here (no GPU): the oracle against the reference's golden
vectors, host logic, and the C-ABI library's exports.  `-m gpu` runs on a
B200 and checks the CUDA path against the oracle and the golden vectors.
"""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); calls the C-ABI kernels")


# features that exist only in the NVRTC-generated kernels (the persistent
# network kernel, the specialised modules): skipped when the generic
# table-driven kernels are forced (HHB_NO_JIT=1 runs of the GPU suite)
requires_jit = pytest.mark.skipif(os.environ.get("HHB_NO_JIT", "0") not in ("", "0"),
                                  reason="JIT-only feature (HHB_NO_JIT set)")


def golden(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False)


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("gpu test run without a CUDA device")
    from paper_2601_21407_b200 import _native
    _native.load()
    return torch.device("cuda", 0)
