"""CPU-side checks of the C-ABI library: it loads and exports every symbol
include/nbx.h declares (no compute calls: there is no GPU here)."""

import re
from pathlib import Path

REPO = Path(__file__).resolve().parents[1]


def declared_symbols():
    text = (REPO / "include" / "nbx.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return set(re.findall(r"\b(nbx_[a-z0-9_]+)\s*\(", text))


def test_library_exports_every_declared_symbol():
    from paper_1506_00716_b200 import _lib

    lib = _lib.load()
    declared = declared_symbols()
    assert declared, "no declarations parsed"
    assert declared == set(_lib.EXPORTS)
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.nbx_version() == 1


def test_library_is_sm100a():
    import subprocess

    so = REPO / "paper_1506_00716_b200" / "libnbx.so"
    out = subprocess.run(["cuobjdump", "--list-elf", str(so)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_package_fails_loudly_without_gpu():
    import pytest
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import numpy as np

    import paper_1506_00716_b200 as nbx

    s = nbx.ParticleSystem(positions=np.zeros((4, 3)), velocities=np.zeros((4, 3)), masses=np.ones(4),
                           charges=np.zeros(4), lj_type=np.zeros(4, dtype=int), box=nbx.SimBox([3.0] * 3))
    with pytest.raises(RuntimeError):
        nbx.build_cluster_grid(s, 4)
