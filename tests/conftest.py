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


LARGE_PREFIXES = ("spc24k_", "spc96k_")


def golden_names():
    """Small fixtures: full reference arrays (grids, lists, forces)."""
    return sorted(p.stem for p in GOLDEN.glob("*.npz")
                  if p.stem not in ("scalars", "diagnostics") and not p.stem.startswith(LARGE_PREFIXES))


def large_golden_names():
    """BASELINE-size fixtures (make_golden.py --large): reference digests of
    the grid and lists, counts, forces and energies."""
    return sorted(p.stem for p in GOLDEN.glob("*.npz") if p.stem.startswith(LARGE_PREFIXES))


def digest(*arrays) -> str:
    """Same digest as tests/golden/make_golden.py:digest."""
    import hashlib

    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype).encode())
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()


def pack_bits(masks) -> np.ndarray:
    masks = np.asarray(masks)
    rows, m, _ = masks.shape
    flat = masks.reshape(rows, m * m).astype(np.uint64)
    w = np.uint64(1) << np.arange(m * m, dtype=np.uint64)
    return (flat * w).sum(axis=1, dtype=np.uint64)


def list_digest(offsets, j_idx, mask_bits) -> str:
    return digest(np.asarray(offsets, dtype=np.int64), np.asarray(j_idx, dtype=np.int64),
                  np.asarray(mask_bits, dtype=np.uint64))


def grid_digest(perm, fill_mask, cell_of_cluster, bboxes) -> str:
    return digest(np.asarray(perm, dtype=np.int64), np.asarray(fill_mask, dtype=np.bool_),
                  np.asarray(cell_of_cluster, dtype=np.int64), np.asarray(bboxes, dtype=np.float64))


def large_system(g):
    """The fixture's SPC box, regenerated and pinned by its digest."""
    from paper_1506_00716_b200.systems import spc_water

    s, table = spc_water(int(g["n"]), seed=int(g["seed"]))
    assert digest(np.asarray(s.positions, dtype=np.float64)) == str(g["positions_digest"])
    occ = None if np.isnan(g["occupancy"]) else float(g["occupancy"])
    return s, table, occ


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
