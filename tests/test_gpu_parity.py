"""GPU parity: the sm_100a path (through the drop-in Python API and the C ABI)
against golden vectors from the reference and against the CPU oracle.

Bars (BASELINE.json north_star): grid and lists bit-identical / set-identical
(indices and masks); forces within 1e-4 relative RMS (FP32 pair math);
energies within 1e-5 relative (FP64 accumulation).
"""

import numpy as np
import pytest

from conftest import golden_names, load_golden

pytestmark = pytest.mark.gpu

FORCE_RTOL = 1e-4   # relative RMS, north_star
ENERGY_RTOL = 1e-5  # relative, north_star

CASES = golden_names()


def _nbx():
    import paper_1506_00716_b200 as nbx

    return nbx


def _system(g):
    nbx = _nbx()
    n = g["positions"].shape[0]
    return nbx.ParticleSystem(positions=g["positions"], velocities=np.zeros((n, 3)),
                              masses=g["masses"], charges=g["charges"], lj_type=g["lj_type"],
                              box=nbx.SimBox(g["box"]))


def _occ(g):
    return None if np.isnan(g["occupancy"]) else float(g["occupancy"])


def rel_rms(f, ref):
    den = float((ref ** 2).sum())
    return float(np.sqrt(((f - ref) ** 2).sum() / den)) if den else float(np.abs(f).max())


def rel(a, b):
    return abs(a - b) / abs(b) if b != 0 else abs(a - b)


@pytest.mark.parametrize("name", CASES)
def test_grid_bit_identical(name):
    nbx = _nbx()
    g = load_golden(name)
    s = _system(g)
    grid = nbx.build_cluster_grid(s, int(g["m"]), _occ(g))
    assert grid.cell_counts == tuple(g["cell_counts"])
    assert grid.n_clusters == g["bboxes"].shape[0]
    for key in ("perm", "inverse_perm", "fill_mask", "cell_of_cluster", "clustered_positions", "bboxes"):
        assert np.array_equal(getattr(grid, key), g[key]), key


@pytest.mark.parametrize("name", CASES)
def test_lists_set_identical(name):
    nbx = _nbx()
    g = load_golden(name)
    s = _system(g)
    grid = nbx.build_cluster_grid(s, int(g["m"]), _occ(g))
    sc = int(g["supercluster"])
    built = nbx.build_pair_list(grid, s.box, float(g["r_list"]), supercluster_size=sc)
    assert np.array_equal(built.offsets, g["built_offsets"])
    assert np.array_equal(built.j_idx, g["built_j"])
    assert np.array_equal(built.mask_bits, g["built_masks"])
    pruned = nbx.prune_pair_list(built, grid.clustered_positions, s.box)
    assert np.array_equal(pruned.offsets, g["pruned_offsets"])
    assert np.array_equal(pruned.j_idx, g["pruned_j"])
    assert np.array_equal(pruned.mask_bits, g["pruned_masks"])
    # prune is idempotent (test_pairlist.py:72-82)
    again = nbx.prune_pair_list(pruned, grid.clustered_positions, s.box)
    assert np.array_equal(again.j_idx, pruned.j_idx) and np.array_equal(again.offsets, pruned.offsets)
    # fused build + prune (one search) is bit-identical to the two steps
    fused = nbx.build_pruned_pair_list(grid, s.box, float(g["r_list"]), supercluster_size=sc)
    assert np.array_equal(fused.offsets, g["pruned_offsets"])
    assert np.array_equal(fused.j_idx, g["pruned_j"])
    assert np.array_equal(fused.mask_bits, g["pruned_masks"])
    stats = nbx.interaction_stats(pruned, grid, grid.clustered_positions, s.box, float(g["r_cut"]))
    assert stats.n_admitted == int(g["n_admitted"])
    assert stats.n_within_cutoff == int(g["n_within"])
    if sc > 1:
        assert np.array_equal(built.super_offsets, g["built_super_offsets"])
        assert np.array_equal(built.super_j_idx, g["built_super_j"])
        assert np.array_equal(built.super_pair_idx, g["built_super_pair_idx"])
        assert np.array_equal(pruned.super_offsets, g["super_offsets"])
        assert np.array_equal(pruned.super_j_idx, g["super_j"])
        assert np.array_equal(pruned.super_pair_idx, g["super_pair_idx"])


def _setup(name):
    nbx = _nbx()
    g = load_golden(name)
    s = _system(g)
    m = int(g["m"])
    params = nbx.NonbondedParams(r_cut=float(g["r_cut"]), r_list=float(g["r_list"]),
                                 lj_table=g["lj_table"], shift_potential=bool(g["shift"]))
    grid = nbx.build_cluster_grid(s, m, _occ(g))
    plist = nbx.prune_pair_list(
        nbx.build_pair_list(grid, s.box, float(g["r_list"]), supercluster_size=int(g["supercluster"])),
        grid.clustered_positions, s.box)
    return nbx, g, s, params, grid, plist, nbx.KernelLayout(m=m, n_lane=m)


@pytest.mark.parametrize("name", CASES)
def test_forces_match_reference(name):
    nbx, g, s, params, grid, plist, layout = _setup(name)
    res = nbx.compute_nonbonded_original(plist, grid, s.positions, s.charges, s.lj_type, params, s.box, layout)
    assert rel_rms(res.forces, g["f_original"]) <= FORCE_RTOL
    assert rel(res.e_lj, float(g["e_lj"])) <= ENERGY_RTOL
    assert rel(res.e_coulomb, float(g["e_coulomb"])) <= ENERGY_RTOL
    # against the reference brute force as well (oracle.py:28-67)
    assert rel_rms(res.forces, g["bf_forces"]) <= FORCE_RTOL
    assert rel(res.e_lj, float(g["bf_e_lj"])) <= ENERGY_RTOL
    assert rel(res.e_coulomb, float(g["bf_e_coulomb"])) <= ENERGY_RTOL
    # clustered order (compute_nonbonded) and the accumulate contract
    rc = nbx.compute_nonbonded(plist, grid, s.positions, s.charges, s.lj_type, params, s.box, layout)
    assert rel_rms(rc.forces, g["f_clustered"]) <= FORCE_RTOL
    f_out = np.ones((grid.n_slots, 3))
    nbx.compute_nonbonded_into(plist, grid, s.positions, s.charges, s.lj_type, params, s.box, layout, f_out)
    assert rel_rms(f_out - 1.0, g["f_clustered"]) <= FORCE_RTOL


@pytest.mark.parametrize("name", ["spc3k_tuned", "uniform_m2", "uniform_m8", "charged_fluid600"])
def test_subsets_sum_to_whole_and_canonical_path(name):
    """i_sel chunks (engine.parallel_forces workers) add up to the full pass;
    the canonical-row kernel agrees with the grouped kernel."""
    nbx, g, s, params, grid, plist, layout = _setup(name)
    full = np.zeros((grid.n_slots, 3))
    e_full = nbx.compute_nonbonded_into(plist, grid, s.positions, s.charges, s.lj_type, params, s.box,
                                        layout, full)
    parts = np.zeros((grid.n_slots, 3))
    e_sum = np.zeros(2)
    n_units = plist.n_super_groups if plist.supercluster_size > 1 else plist.n_i_clusters
    for chunk in np.array_split(np.arange(n_units), 3):
        e = nbx.compute_nonbonded_into(plist, grid, s.positions, s.charges, s.lj_type, params, s.box,
                                       layout, parts, i_sel=chunk)
        e_sum += e
    assert rel_rms(parts, full) <= FORCE_RTOL  # grouped vs canonical kernel: FP32 rounding only
    # FP32 per-pair energies grouped differently: FP32-level agreement
    assert rel(e_sum[0], e_full[0]) <= ENERGY_RTOL and rel(e_sum[1], e_full[1]) <= ENERGY_RTOL


def test_bit_reproducible_reruns():
    nbx, g, s, params, grid, plist, layout = _setup("spc3k_default")
    a = nbx.compute_nonbonded_original(plist, grid, s.positions, s.charges, s.lj_type, params, s.box, layout)
    b = nbx.compute_nonbonded_original(plist, grid, s.positions, s.charges, s.lj_type, params, s.box, layout)
    assert np.array_equal(a.forces, b.forces)
    assert a.e_lj == b.e_lj and a.e_coulomb == b.e_coulomb


def test_singular_pair_reports_original_indices():
    nbx = _nbx()
    pos = np.array([[1.0, 1.0, 1.0], [2.0, 2.0, 2.0], [1.0, 1.0, 1.0], [3.0, 1.5, 2.5]])
    s = nbx.ParticleSystem(positions=pos, velocities=np.zeros((4, 3)), masses=np.ones(4),
                           charges=np.zeros(4), lj_type=np.zeros(4, dtype=int), box=nbx.SimBox([5.0] * 3))
    params = nbx.NonbondedParams(r_cut=0.9, r_list=1.0, lj_table=[[[1.0, 0.3]]])
    grid = nbx.build_cluster_grid(s, 1)
    plist = nbx.build_pair_list(grid, s.box, 1.0)
    with pytest.raises(nbx.SingularityError) as err:
        nbx.compute_nonbonded_original(plist, grid, s.positions, s.charges, s.lj_type, params, s.box,
                                       nbx.KernelLayout(1, 1))
    assert {err.value.i, err.value.j} == {0, 2}


def test_parameter_errors():
    nbx = _nbx()
    g = load_golden("uniform_m4")
    s = _system(g)
    with pytest.raises(nbx.ParameterError):
        nbx.build_cluster_grid(s, 3)
    grid = nbx.build_cluster_grid(s, 4)
    with pytest.raises(nbx.ParameterError):
        nbx.build_pair_list(grid, s.box, 2.0)       # box edge < 2 r_list
    with pytest.raises(nbx.ParameterError):
        nbx.build_pair_list(grid, s.box, 0.0)
    with pytest.raises(nbx.ParameterError):
        nbx.build_pair_list(grid, s.box, 1.0, supercluster_size=4)
    plist = nbx.build_pair_list(grid, s.box, 1.0)
    with pytest.raises(nbx.ParameterError):
        nbx.prune_pair_list(plist, np.zeros((3, 3)), s.box)


def test_empty_system():
    nbx = _nbx()
    s = nbx.ParticleSystem(positions=np.zeros((0, 3)), velocities=np.zeros((0, 3)), masses=np.zeros(0),
                           charges=np.zeros(0), lj_type=np.zeros(0, dtype=int), box=nbx.SimBox([3.0] * 3))
    grid = nbx.build_cluster_grid(s, 4)
    assert grid.n_clusters == 0 and grid.perm.shape == (0,)
    plist = nbx.build_pair_list(grid, s.box, 1.0)
    assert plist.n_pairs == 0


# ---------------------------------------------------------------- larger sizes vs the C oracle
def _spc(n, occ_rule):
    nbx = _nbx()
    from paper_1506_00716_b200.systems import spc_water, tuned_occupancy

    s, table = spc_water(n, seed=2024)
    occ = tuned_occupancy(n, float(s.box.lengths[0]), 4) if occ_rule == "tuned" else None
    return nbx, s, table, occ


@pytest.mark.parametrize("occ_rule", ["default", "tuned"])
def test_spc24k_lists_and_forces_vs_oracle(occ_rule):
    from oracle import forces as of
    from oracle import native, search

    nbx, s, table, occ = _spc(24000, occ_rule)
    L = s.box.lengths
    grid = nbx.build_cluster_grid(s, 4, occ)
    og = search.build_grid(s.positions, L, 4, occ)
    assert np.array_equal(grid.perm, og["perm"]) and np.array_equal(grid.bboxes, og["bboxes"])
    built = nbx.build_pair_list(grid, s.box, 1.1)
    ob = native.search_list(og, L, 1.1)
    assert np.array_equal(built.offsets, ob["offsets"]) and np.array_equal(built.j_idx, ob["j_idx"])
    pruned = nbx.prune_pair_list(built, grid.clustered_positions, s.box)
    op = native.prune_list(ob, og["clustered_positions"], L)
    assert np.array_equal(pruned.offsets, op["offsets"]) and np.array_equal(pruned.j_idx, op["j_idx"])
    assert np.array_equal(pruned.mask_bits, search.pack_masks(op["masks"]))
    fused = nbx.build_pruned_pair_list(grid, s.box, 1.1)
    assert np.array_equal(fused.offsets, op["offsets"]) and np.array_equal(fused.j_idx, op["j_idx"])
    assert np.array_equal(fused.mask_bits, search.pack_masks(op["masks"]))
    layout = nbx.KernelLayout(4, 4)
    for phys, params in (
        (of.Physics(r_cut=1.0, lj_table=table, shift_potential=True),
         nbx.NonbondedParams(r_cut=1.0, r_list=1.1, lj_table=table, shift_potential=True)),
        (of.Physics(r_cut=1.0, lj_table=table, elec="reaction_field", epsilon_rf=0.0),
         nbx.NonbondedParams(r_cut=1.0, r_list=1.1, lj_table=table, elec="reaction_field", epsilon_rf=0.0)),
        (of.Physics(r_cut=1.0, lj_table=table, shift_potential=True, elec="ewald", ewald_beta=of.ewald_beta_for(1.0)),
         nbx.NonbondedParams(r_cut=1.0, r_list=1.1, lj_table=table, shift_potential=True, elec="ewald",
                             ewald_beta=nbx.ewald_beta(1.0))),
    ):
        res = nbx.compute_nonbonded_original(pruned, grid, s.positions, s.charges, s.lj_type, params, s.box, layout)
        fc, elj, ec = native.list_forces(op, og, s.positions, s.charges, s.lj_type, L, phys)
        fref = search.scatter_to_original(og, fc)
        assert rel_rms(res.forces, fref) <= FORCE_RTOL, params.elec
        assert rel(res.e_lj, elj) <= ENERGY_RTOL, params.elec
        assert rel(res.e_coulomb, ec) <= ENERGY_RTOL, params.elec


def test_moved_positions_use_current_coordinates():
    """Force at positions displaced within the buffer (and wrapped across the
    boundary) equals the oracle on the same list (kernels.py: positions are
    gathered per call, minimum image per pair)."""
    from oracle import forces as of
    from oracle import native, search

    nbx, s, table, occ = _spc(3000, "tuned")
    L = s.box.lengths
    grid = nbx.build_cluster_grid(s, 4, occ)
    plist = nbx.prune_pair_list(nbx.build_pair_list(grid, s.box, 1.1), grid.clustered_positions, s.box)
    rng = np.random.default_rng(5)
    step = rng.normal(size=(s.n, 3))
    step *= 0.04 / np.linalg.norm(step, axis=1, keepdims=True)
    moved = s.positions + step
    moved[:50] += L  # an unwrapped image must not matter
    params = nbx.NonbondedParams(r_cut=1.0, r_list=1.1, lj_table=table, shift_potential=True)
    res = nbx.compute_nonbonded_original(plist, grid, moved, s.charges, s.lj_type, params, s.box,
                                         nbx.KernelLayout(4, 4))
    og = search.build_grid(s.positions, L, 4, occ)
    ol = dict(m=4, offsets=plist.offsets, j_idx=plist.j_idx, masks=plist.masks, r_list=1.1)
    fc, elj, ec = native.list_forces(ol, og, moved, s.charges, s.lj_type, L,
                                     of.Physics(r_cut=1.0, lj_table=table, shift_potential=True))
    assert rel_rms(res.forces, search.scatter_to_original(og, fc)) <= FORCE_RTOL
    assert rel(res.e_lj, elj) <= ENERGY_RTOL and rel(res.e_coulomb, ec) <= ENERGY_RTOL


def test_spc96k_bench_config_vs_oracle():
    """BASELINE config 3 (the bench workload): 96k SPC, tuned grid, LJ + Ewald
    real space -- grid and pruned list identical to the oracle's C port,
    forces / energies within the north_star tolerances."""
    from oracle import forces as of
    from oracle import native, search

    nbx, s, table, occ = _spc(96000, "tuned")
    L = s.box.lengths
    grid = nbx.build_cluster_grid(s, 4, occ)
    og = search.build_grid(s.positions, L, 4, occ)
    assert np.array_equal(grid.perm, og["perm"]) and np.array_equal(grid.bboxes, og["bboxes"])
    pruned = nbx.prune_pair_list(nbx.build_pair_list(grid, s.box, 1.1), grid.clustered_positions_device, s.box)
    op = native.prune_list(native.search_list(og, L, 1.1), og["clustered_positions"], L)
    assert np.array_equal(pruned.offsets, op["offsets"]) and np.array_equal(pruned.j_idx, op["j_idx"])
    assert np.array_equal(pruned.mask_bits, search.pack_masks(op["masks"]))
    beta = nbx.ewald_beta(1.0)
    params = nbx.NonbondedParams(r_cut=1.0, r_list=1.1, lj_table=table, shift_potential=True, elec="ewald",
                                 ewald_beta=beta)
    phys = of.Physics(r_cut=1.0, lj_table=table, shift_potential=True, elec="ewald", ewald_beta=beta)
    res = nbx.compute_nonbonded_original(pruned, grid, s.positions, s.charges, s.lj_type, params, s.box,
                                         nbx.KernelLayout(4, 4))
    fc, elj, ec = native.list_forces(op, og, s.positions, s.charges, s.lj_type, L, phys)
    fref = search.scatter_to_original(og, fc)
    assert rel_rms(res.forces, fref) <= FORCE_RTOL
    assert rel(res.e_lj, elj) <= ENERGY_RTOL and rel(res.e_coulomb, ec) <= ENERGY_RTOL


def test_spc1p5m_forces_vs_oracle_and_newton():
    """BASELINE config 4 size (1.5M atoms) on one GPU: forces on the GPU list
    against the oracle's C force pass over the same list, and the
    size-independent property sum_i F_i = 0 (every pair enters twice with
    opposite sign)."""
    from oracle import forces as of
    from oracle import native, search

    nbx, s, table, occ = _spc(1500000, "tuned")
    L = s.box.lengths
    grid = nbx.build_cluster_grid(s, 4, occ)
    pruned = nbx.prune_pair_list(nbx.build_pair_list(grid, s.box, 1.1), grid.clustered_positions_device, s.box)
    beta = nbx.ewald_beta(1.0)
    params = nbx.NonbondedParams(r_cut=1.0, r_list=1.1, lj_table=table, shift_potential=True, elec="ewald",
                                 ewald_beta=beta)
    res = nbx.compute_nonbonded_original(pruned, grid, s.positions, s.charges, s.lj_type, params, s.box,
                                         nbx.KernelLayout(4, 4))
    net = np.abs(res.forces.sum(axis=0)).max()
    assert net <= 1e-6 * np.abs(res.forces).sum(axis=0).max()
    og = search.build_grid(s.positions, L, 4, occ)
    assert np.array_equal(grid.perm, og["perm"])
    ol = dict(m=4, offsets=pruned.offsets, j_idx=pruned.j_idx, masks=pruned.masks, r_list=1.1)
    phys = of.Physics(r_cut=1.0, lj_table=table, shift_potential=True, elec="ewald", ewald_beta=beta)
    fc, elj, ec = native.list_forces(ol, og, s.positions, s.charges, s.lj_type, L, phys)
    fref = search.scatter_to_original(og, fc)
    assert rel_rms(res.forces, fref) <= FORCE_RTOL
    assert rel(res.e_lj, elj) <= ENERGY_RTOL and rel(res.e_coulomb, ec) <= ENERGY_RTOL
