import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def golden(name):
    import numpy as np

    return np.load(os.path.join(GOLDEN, f"{name}.npz"), allow_pickle=False)


@pytest.fixture(scope="session")
def gold():
    return golden


@pytest.fixture(params=["fused", "split"])
def select_path(request):
    """Run a decode test on both selection paths: the fused score/select/
    attend kernel (lrqk_score_attend, the default) and the split one
    (lrqk_score + lrqk_select_attend)."""
    from paper_2510_23649_b200 import _lib

    lib = _lib.lib()
    prev = lib.lrqk_set_fused(1 if request.param == "fused" else 0)
    yield request.param
    lib.lrqk_set_fused(prev)
