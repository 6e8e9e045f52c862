import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))

GOLDEN = Path(__file__).resolve().parent / "golden" / "golden.npz"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu on the GPU box)")


@pytest.fixture(scope="session")
def golden():
    with np.load(GOLDEN) as g:
        return {k: g[k] for k in g.files}


@pytest.fixture(scope="session")
def built_lib():
    """Build libotf_b200.so if stale (nvcc cross-compiles without a GPU)."""
    from paper_1407_4764_b200 import _build

    return _build.build()


@pytest.fixture(scope="session")
def otf(built_lib):
    """The product package on a GPU (gpu tests only)."""
    import paper_1407_4764_b200 as otf

    otf._lib.load(require_device=True)
    return otf
