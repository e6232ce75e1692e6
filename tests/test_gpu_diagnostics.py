"""Diagnostics row on the GPU against the real reference:
write_pairs_csv byte-identical (pairlist.py:349-376; distances from the
device kernel nbx_list_diagnostics), flop_count equal for every n_lane
(kernels.py:443-473), and the device scatter_to_original
(nbx_scatter_to_original, gridder.py:149-162) equal to the reference's
scatter.  Goldens: tests/golden/diagnostics.npz (make_golden.py
--diagnostics)."""

import hashlib

import numpy as np
import pytest

from conftest import GOLDEN, load_golden

pytestmark = pytest.mark.gpu

CASES = [("spc3k_tuned", 4), ("spc3k_default", 4), ("uniform_m8", 8), ("uniform_m2", 2), ("uniform_super8", 4)]


def _diag():
    with np.load(GOLDEN / "diagnostics.npz") as z:
        return {k: z[k] for k in z.files}


def _setup(name, m):
    import paper_1506_00716_b200 as nbx

    g = load_golden(name)
    n = g["positions"].shape[0]
    s = nbx.ParticleSystem(positions=g["positions"], velocities=np.zeros((n, 3)), masses=g["masses"],
                           charges=g["charges"], lj_type=g["lj_type"], box=nbx.SimBox(g["box"]))
    occ = None if np.isnan(g["occupancy"]) else float(g["occupancy"])
    grid = nbx.build_cluster_grid(s, m, occ)
    built = nbx.build_pair_list(grid, s.box, float(g["r_list"]), supercluster_size=int(g["supercluster"]))
    pruned = nbx.prune_pair_list(built, grid.clustered_positions, s.box)
    return nbx, g, s, grid, built, pruned


@pytest.mark.parametrize("name,m", CASES)
def test_write_pairs_csv_byte_identical(name, m, tmp_path):
    nbx, g, s, grid, built, pruned = _setup(name, m)
    d = _diag()
    for tag, pl in (("built", built), ("pruned", pruned)):
        path = tmp_path / f"{tag}.csv"
        nbx.write_pairs_csv(pl, grid, s.box, path)
        assert hashlib.sha256(path.read_bytes()).hexdigest() == str(d[f"{name}_{tag}_csv_sha256"]), tag


@pytest.mark.parametrize("name,m", CASES)
def test_flop_count_matches_reference(name, m):
    nbx, g, s, grid, built, pruned = _setup(name, m)
    d = _diag()
    for nl, total, useful in d[f"{name}_flops"]:
        fc = nbx.flop_count(pruned, grid, nbx.KernelLayout(m=m, n_lane=int(nl)), s.box, float(g["r_cut"]))
        assert fc.total_flops == int(total) and fc.useful_flops == int(useful), nl


@pytest.mark.parametrize("name,m", CASES)
def test_device_scatter_to_original(name, m):
    import torch

    nbx, g, s, grid, built, pruned = _setup(name, m)
    d = _diag()
    vin = torch.as_tensor(d[f"{name}_scatter_in"], device="cuda")
    out = nbx.scatter_to_original(grid, vin)
    assert out.is_cuda
    assert np.array_equal(out.cpu().numpy(), d[f"{name}_scatter_out"])
    # one column (k = 1) and the host path agree too
    out1 = nbx.scatter_to_original(grid, vin[:, 1].contiguous())
    assert np.array_equal(out1.cpu().numpy(), d[f"{name}_scatter_out"][:, 1])
    assert np.array_equal(nbx.scatter_to_original(grid, d[f"{name}_scatter_in"]), d[f"{name}_scatter_out"])
