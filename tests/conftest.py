import os
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA path)")
    config.addinivalue_line("markers", "slow: long-running parity case")


def _have_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


HAVE_GPU = _have_gpu()


def pytest_collection_modifyitems(config, items):
    if HAVE_GPU:
        return
    skip = pytest.mark.skip(reason="no GPU in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def oracle_ref():
    """The compiled reference (oracle/_ref); built here when /root/reference exists."""
    from oracle import ref
    if not ref.available() and Path("/root/reference/proj").exists():
        ref.build()
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    return ref


@pytest.fixture(scope="session")
def mlg():
    import paper_1401_4969_b200 as m
    m.lib()  # fails loudly if the CUDA library is missing
    return m
