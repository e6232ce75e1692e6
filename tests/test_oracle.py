"""Pin the CPU oracle against golden vectors produced by the real reference.

The oracle (oracle/) is the checker for every GPU parity test, so it must
reproduce the reference bit for bit where the reference is deterministic
(grid, lists, prune, admitted/within counts) and to ~1e-12 for forces.
"""

import numpy as np
import pytest

from conftest import golden_names, load_golden
from oracle import forces as of
from oracle import native, search
from oracle.geometry import min_image, wrap

CASES = golden_names()


def _grid(g):
    occ = None if np.isnan(g["occupancy"]) else float(g["occupancy"])
    return search.build_grid(g["positions"], g["box"], int(g["m"]), occ)


def _phys(g):
    return of.Physics(r_cut=float(g["r_cut"]), lj_table=g["lj_table"], shift_potential=bool(g["shift"]))


@pytest.mark.parametrize("name", CASES)
def test_grid_bit_identical(name):
    g = load_golden(name)
    grid = _grid(g)
    assert np.array_equal(grid["perm"], g["perm"])
    assert np.array_equal(grid["inverse_perm"], g["inverse_perm"])
    assert np.array_equal(grid["fill_mask"], g["fill_mask"])
    assert np.array_equal(grid["cell_of_cluster"], g["cell_of_cluster"])
    assert (grid["cells"], grid["cells"]) == tuple(g["cell_counts"])
    assert np.array_equal(grid["clustered_positions"], g["clustered_positions"])
    assert np.array_equal(grid["bboxes"], g["bboxes"])


@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("method", ["numpy", "n2", "cols"])
def test_search_and_prune_bit_identical(name, method):
    g = load_golden(name)
    grid = _grid(g)
    if method == "numpy":
        built = search.build_pairs_bruteforce(grid, g["box"], float(g["r_list"]))
        pruned = search.prune(built, grid["clustered_positions"], g["box"])
    else:
        built = native.search_list(grid, g["box"], float(g["r_list"]), method=method)
        pruned = native.prune_list(built, grid["clustered_positions"], g["box"])
    assert np.array_equal(built["offsets"], g["built_offsets"])
    assert np.array_equal(built["j_idx"], g["built_j"])
    assert np.array_equal(search.pack_masks(built["masks"]), g["built_masks"])
    assert np.array_equal(pruned["offsets"], g["pruned_offsets"])
    assert np.array_equal(pruned["j_idx"], g["pruned_j"])
    assert np.array_equal(search.pack_masks(pruned["masks"]), g["pruned_masks"])


@pytest.mark.parametrize("name", CASES)
def test_counts_and_super_layout(name):
    g = load_golden(name)
    grid = _grid(g)
    lst = dict(m=int(g["m"]), offsets=g["pruned_offsets"], j_idx=g["pruned_j"].astype(np.int64),
               masks=search.unpack_masks(g["pruned_masks"], int(g["m"])), r_list=float(g["r_list"]))
    assert int(lst["masks"].sum()) == int(g["n_admitted"])
    assert search.count_within(lst, grid["clustered_positions"], g["box"], float(g["r_cut"])) == int(g["n_within"])
    assert native.count_within(lst, grid["clustered_positions"], g["box"], float(g["r_cut"])) == int(g["n_within"])
    if int(g["supercluster"]) > 1:
        so, sj, sp = search.super_layout(lst["offsets"], lst["j_idx"], grid["n_clusters"], 8)
        assert np.array_equal(so, g["super_offsets"])
        assert np.array_equal(sj, g["super_j"])
        assert np.array_equal(sp, g["super_pair_idx"])
        so, sj, sp = search.super_layout(g["built_offsets"], g["built_j"].astype(np.int64), grid["n_clusters"], 8)
        assert np.array_equal(so, g["built_super_offsets"])
        assert np.array_equal(sp, g["built_super_pair_idx"])


@pytest.mark.parametrize("name", CASES)
def test_forces_match_reference(name):
    g = load_golden(name)
    grid = _grid(g)
    lst = dict(m=int(g["m"]), offsets=g["pruned_offsets"], j_idx=g["pruned_j"].astype(np.int64),
               masks=search.unpack_masks(g["pruned_masks"], int(g["m"])), r_list=float(g["r_list"]))
    phys = _phys(g)
    scale = np.abs(g["f_clustered"]).max()
    for fc, elj, ec in (
        native.list_forces(lst, grid, g["positions"], g["charges"], g["lj_type"], g["box"], phys, threads=1),
        native.list_forces(lst, grid, g["positions"], g["charges"], g["lj_type"], g["box"], phys, threads=3),
        of.list_forces(lst, grid, g["positions"], g["charges"], g["lj_type"], g["box"], phys),
    ):
        assert np.abs(fc - g["f_clustered"]).max() <= 1e-12 * scale
        assert abs(elj - float(g["e_lj"])) <= 1e-12 * max(1.0, abs(float(g["e_lj"])))
        assert abs(ec - float(g["e_coulomb"])) <= 1e-12 * max(1.0, abs(float(g["e_coulomb"])))
    fo = search.scatter_to_original(grid, fc)
    assert np.abs(fo - g["f_original"]).max() <= 1e-12 * scale


def test_native_force_threads_bit_reproducible():
    g = load_golden("spc3k_tuned")
    grid = _grid(g)
    lst = dict(m=4, offsets=g["pruned_offsets"], j_idx=g["pruned_j"].astype(np.int64),
               masks=search.unpack_masks(g["pruned_masks"], 4), r_list=1.1)
    phys = _phys(g)
    a = native.list_forces(lst, grid, g["positions"], g["charges"], g["lj_type"], g["box"], phys, threads=4)
    b = native.list_forces(lst, grid, g["positions"], g["charges"], g["lj_type"], g["box"], phys, threads=4)
    assert np.array_equal(a[0], b[0]) and a[1] == b[1] and a[2] == b[2]


@pytest.mark.parametrize("name", ["spc3k_tuned", "uniform_m4", "charged_fluid600"])
def test_brute_force_matches_reference(name):
    g = load_golden(name)
    if name.startswith("spc3k"):
        pytest.skip("3k brute force covered via list forces; keep the CPU suite fast")
    f, elj, ec = of.brute_force(g["positions"], g["charges"], g["lj_type"], g["box"], _phys(g))
    scale = np.abs(g["bf_forces"]).max()
    assert np.abs(f - g["bf_forces"]).max() <= 1e-12 * scale
    assert abs(elj - float(g["bf_e_lj"])) <= 1e-12 * max(1.0, abs(float(g["bf_e_lj"])))
    assert abs(ec - float(g["bf_e_coulomb"])) <= 1e-12 * max(1.0, abs(float(g["bf_e_coulomb"])))


def test_known_answers():
    z = np.load(__import__("conftest").GOLDEN / "scalars.npz")
    phys = of.Physics(r_cut=0.9, lj_table=np.array([[[0.0, 0.3]]]))
    e_lj, e_c, fr = of.pair_terms(0.25, 0, 0, 1.0, -1.0, phys)
    assert float(e_lj + e_c) == float(z["coulomb_e"])
    assert float(fr) == float(z["coulomb_fr"])
    assert float(e_lj + e_c) == pytest.approx(-277.870916, rel=1e-12)  # test_kernels.py:27-33
    pos = np.zeros((6, 3))
    pos[:, 2] = [0.5, 0.5, 0.5, 0.2, 0.2, 0.9]
    grid = search.build_grid(pos, [2.0, 2.0, 2.0], 2, 1000)
    assert grid["perm"].tolist() == [3, 4, 0, 1, 2, 5] == z["tie_perm"].tolist()


def test_geometry_edges():
    L = np.array([2.0, 3.0, 4.0])
    assert np.array_equal(wrap(wrap(np.array([[-1e-17, 2.0, -4.0]]), L), L), wrap(np.array([[-1e-17, 2.0, -4.0]]), L))
    assert np.all(wrap(np.array([[-1e-17, 2.0, -4.0]]), L) < L)
    assert min_image(np.array([-1.0, 1.5, 2.0]), L).tolist() == [-1.0, -1.5, -2.0]


def test_rf_eps1_equals_shifted_cutoff_and_ewald_dimer():
    tab = np.array([[[0.65, 0.3166]]])
    cut = of.Physics(r_cut=1.0, lj_table=tab, shift_potential=True)
    rf1 = of.Physics(r_cut=1.0, lj_table=tab, shift_potential=True, elec="reaction_field", epsilon_rf=1.0)
    r2 = np.linspace(0.05, 1.0, 50)
    a = of.pair_terms(r2, 0, 0, 0.41, -0.82, cut)
    b = of.pair_terms(r2, 0, 0, 0.41, -0.82, rf1)
    for x, y in zip(a, b):
        np.testing.assert_allclose(x, y, rtol=1e-13, atol=1e-13)
    beta = of.ewald_beta_for(1.0)
    from scipy.special import erfc
    assert erfc(beta) == pytest.approx(1e-5, rel=1e-9)
    ew = of.Physics(r_cut=1.0, lj_table=np.array([[[0.0, 0.3]]]), elec="ewald", ewald_beta=beta)
    # F/r from a numerical derivative of the energy
    r = 0.37
    h = 1e-6
    e = lambda rr: float(of.pair_terms(rr * rr, 0, 0, 1.0, 1.0, ew)[1])
    fnum = -(e(r + h) - e(r - h)) / (2 * h) / r
    assert float(of.pair_terms(r * r, 0, 0, 1.0, 1.0, ew)[2]) == pytest.approx(fnum, rel=1e-7)


# ---------------------------------------------------------------- BASELINE sizes (24k / 96k)
from conftest import digest, grid_digest, large_golden_names, large_system, list_digest  # noqa: E402


@pytest.mark.parametrize("name", large_golden_names())
def test_large_fixture_oracle(name):
    """The oracle's C port reproduces the reference at the BASELINE sizes:
    grid and built / pruned lists bit-identical (SHA-256 of the reference's
    arrays), admitted / within counts equal, forces to FP64 rounding."""
    g = load_golden(name)
    s, table, occ = large_system(g)
    L = s.box.lengths
    m = int(g["m"])
    grid = search.build_grid(s.positions, L, m, occ)
    assert grid_digest(grid["perm"], grid["fill_mask"], grid["cell_of_cluster"], grid["bboxes"]) == str(g["grid_digest"])
    built = native.search_list(grid, L, float(g["r_list"]), method="cols")
    assert list_digest(built["offsets"], built["j_idx"], search.pack_masks(built["masks"])) == str(g["built_digest"])
    pruned = native.prune_list(built, grid["clustered_positions"], L)
    assert list_digest(pruned["offsets"], pruned["j_idx"], search.pack_masks(pruned["masks"])) == \
        str(g["pruned_digest"])
    assert int(search.unpack_masks(search.pack_masks(pruned["masks"]), m).sum()) == int(g["n_admitted"])
    assert native.count_within(pruned, grid["clustered_positions"], L, float(g["r_cut"])) == int(g["n_within"])
    phys = of.Physics(r_cut=float(g["r_cut"]), lj_table=table, shift_potential=bool(g["shift"]))
    fc, elj, ec = native.list_forces(pruned, grid, s.positions, s.charges, s.lj_type, L, phys)
    f = search.scatter_to_original(grid, fc)
    ref = g["f_original"].astype(np.float64)
    tol = 1e-12 if g["f_original"].dtype == np.float64 else 1e-6  # 96k fixtures store FP32 forces
    assert np.sqrt(((f - ref) ** 2).sum() / (ref ** 2).sum()) <= tol
    assert abs(elj - float(g["e_lj"])) <= 1e-12 * abs(float(g["e_lj"]))
    assert abs(ec - float(g["e_coulomb"])) <= 1e-12 * abs(float(g["e_coulomb"]))
