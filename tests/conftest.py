import os
import sys
from pathlib import Path

import numpy as np
import pytest

REPO = Path(__file__).resolve().parents[1]
GOLDEN = REPO / "tests" / "golden"
sys.path.insert(0, str(REPO))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: large sizes; minutes of CPU or GPU time")


def golden_names():
    return sorted(p.stem for p in GOLDEN.glob("*.npz") if p.stem != "scalars")


def load_golden(name):
    with np.load(GOLDEN / f"{name}.npz") as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def have_gpu():
    import torch

    return torch.cuda.is_available()


def pytest_collection_modifyitems(config, items):
    try:
        import torch

        gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        gpu = False
    if gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
