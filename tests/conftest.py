import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "slow: long-running")


def has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


@pytest.fixture(scope="session")
def grids_golden():
    return np.load(os.path.join(GOLDEN, "grids.npz"))


@pytest.fixture(scope="session")
def runmaps_golden():
    return np.load(os.path.join(GOLDEN, "runmaps.npz"))


@pytest.fixture(scope="session")
def goal_views_golden():
    return np.load(os.path.join(GOLDEN, "goal_views.npz"))


@pytest.fixture(scope="session")
def ctx():
    """A product context on cuda:0 (GPU tests only)."""
    import ctypes as C

    from paper_1909_07717_b200 import abi
    lib = abi.load_library()
    h = C.c_void_p()
    st = lib.pp_ctx_create(0, C.byref(h))
    assert st == 0, f"pp_ctx_create failed: {st}"
    yield h
    lib.pp_ctx_destroy(h)
