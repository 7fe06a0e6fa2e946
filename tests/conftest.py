import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA library)")
    config.addinivalue_line("markers", "slow: long-running parity case")


def _has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


@pytest.fixture(scope="session")
def oracle():
    """The reference library built from /root/reference against the Eigen shim."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import ref  # noqa: E402
    if not ref.available():
        ref.build()
    if not ref.available():
        pytest.skip("oracle/_ref not built and /root/reference absent")
    return ref.load()


@pytest.fixture(scope="session")
def b200():
    """The product library on cuda:0. Fails (not skips) when unbuilt."""
    from paper_2112_00821_b200 import Backend
    if not _has_gpu():
        pytest.skip("no GPU in this container")
    return Backend.b200()


@pytest.fixture(scope="session")
def b200_host():
    """The product library loaded without a GPU (host-side geometry only)."""
    from paper_2112_00821_b200 import Backend
    path = os.path.join(ROOT, "paper_2112_00821_b200", "_lib", "libfmvs.so")
    if not os.path.exists(path):
        raise RuntimeError("libfmvs.so not built: run __graft_entry__.build()")
    return Backend(path, "fmvs_", needs_context=False)


@pytest.fixture
def rng():
    return np.random.default_rng(12345)
