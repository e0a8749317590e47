import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests through the C-ABI")
    config.addinivalue_line("markers", "slow: long-running (full-size configs)")


def pytest_sessionstart(session):
    # a fresh checkout has no libsketchmp.so (build output, git-ignored): cross-compile it once
    # (nvcc needs no GPU); the ABI tests then load it, and -m gpu runs use the same in-tree build
    lib = os.path.join(ROOT, "paper_2311_03393_b200", "libsketchmp.so")
    if not os.path.exists(lib) and not os.environ.get("SKMP_LIB"):
        from paper_2311_03393_b200 import build
        build.build()


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("no CUDA device: -m gpu tests must run on a B200 (no CPU fallback)")
    import paper_2311_03393_b200 as skmp
    skmp.lib()  # fails loudly when the extension is missing
    return torch.device("cuda:0")
