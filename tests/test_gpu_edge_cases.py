"""Edge cases of the reference's own test suite, run through the GPU path and
compared with the oracle (itself pinned to the reference): a single
particle, z ties in a column, a pair exactly at r_c, tiny negative and
exactly-L coordinates, half-box separations, Newton's third law, isolated
particles (reference tests: test_gridder.py single_particle_grid,
z_ties_break_by_original_index; test_kernels.py pair_exactly_at_cutoff_is_
included, beyond_cutoff_admitted_pairs_contribute_nothing, forces_sum_to_zero;
test_model.py wrap_tiny_negative, minimum_image_half_box_boundary;
test_pairlist.py interaction_stats_two_isolated_particles)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

def _table():
    from paper_1506_00716_b200.systems import spc_water

    return spc_water(30)[1]  # the SPC (epsilon, sigma) table; type 0 = O


def _nbx():
    import paper_1506_00716_b200 as nbx

    return nbx


def _system(pos, L, q=None, t=None):
    nbx = _nbx()
    pos = np.asarray(pos, dtype=np.float64).reshape(-1, 3)
    n = pos.shape[0]
    return nbx.ParticleSystem(positions=pos, velocities=np.zeros((n, 3)), masses=np.ones(n),
                              charges=np.zeros(n) if q is None else np.asarray(q, dtype=np.float64),
                              lj_type=np.zeros(n, dtype=np.int64) if t is None else np.asarray(t, dtype=np.int64),
                              box=nbx.SimBox(np.asarray(L, dtype=np.float64)))


def _vs_oracle(s, m, r_list, params, phys, occ=None):
    """GPU grid, lists, forces and energies against the oracle on the same inputs."""
    from oracle import native, search

    nbx = _nbx()
    L = s.box.lengths
    grid = nbx.build_cluster_grid(s, m, occ)
    og = search.build_grid(s.positions, L, m, occ)
    for key in ("perm", "fill_mask", "cell_of_cluster", "clustered_positions", "bboxes"):
        assert np.array_equal(getattr(grid, key), og[key]), key
    built = nbx.build_pair_list(grid, s.box, r_list)
    ob = native.search_list(og, L, r_list)
    assert np.array_equal(built.offsets, ob["offsets"]) and np.array_equal(built.j_idx, ob["j_idx"])
    pruned = nbx.prune_pair_list(built, grid.clustered_positions, s.box)
    op = native.prune_list(ob, og["clustered_positions"], L)
    assert np.array_equal(pruned.offsets, op["offsets"]) and np.array_equal(pruned.j_idx, op["j_idx"])
    assert np.array_equal(pruned.mask_bits, search.pack_masks(op["masks"]))
    res = nbx.compute_nonbonded_original(pruned, grid, s.positions, s.charges, s.lj_type, params, s.box,
                                         nbx.KernelLayout(m, m))
    fc, elj, ec = native.list_forces(op, og, s.positions, s.charges, s.lj_type, L, phys)
    fref = search.scatter_to_original(og, fc)
    return res, fref, elj, ec, pruned, grid


def _cutoff_physics(r_cut=1.0):
    from oracle import forces as of

    nbx = _nbx()
    return (nbx.NonbondedParams(r_cut=r_cut, r_list=r_cut + 0.1, lj_table=_table(), shift_potential=True),
            of.Physics(r_cut=r_cut, lj_table=_table(), shift_potential=True))


@pytest.mark.parametrize("m", [1, 2, 4, 8])
def test_single_particle(m):
    s = _system([[0.3, 2.9, 1.7]], [3.0, 3.0, 3.0], q=[0.5])
    params, phys = _cutoff_physics()
    res, fref, elj, ec, pruned, grid = _vs_oracle(s, m, 1.1, params, phys)
    assert grid.n_clusters == 1 and grid.fill_mask.sum() == m - 1
    assert pruned.n_pairs == 1 and not pruned.masks.any()  # the self row, nothing admitted
    assert np.array_equal(res.forces, np.zeros((1, 3))) and res.e_lj == 0.0 and res.e_coulomb == 0.0


def test_z_ties_break_by_original_index():
    # one column, equal z for several particles: (z, index) order as lexsort
    pos = [[0.5, 0.5, 1.0], [0.6, 0.4, 0.5], [0.4, 0.6, 1.0], [0.5, 0.5, 0.5], [0.55, 0.45, 1.0]]
    s = _system(pos, [4.0, 4.0, 4.0])
    nbx = _nbx()
    grid = nbx.build_cluster_grid(s, 2, 100.0)  # one cell
    assert grid.cell_counts == (1, 1)
    real = grid.perm[~grid.fill_mask]
    assert real.tolist() == [1, 3, 0, 2, 4]
    params, phys = _cutoff_physics()
    _vs_oracle(s, 2, 1.1, params, phys, occ=100.0)


def test_pair_exactly_at_cutoff_is_included():
    nbx = _nbx()
    params, phys = _cutoff_physics(1.0)
    L = [5.0, 5.0, 5.0]
    at = _system([[1.0, 1.0, 1.0], [2.0, 1.0, 1.0]], L, q=[0.4, -0.4])  # |dx| == 1.0 exactly in FP64
    res, fref, elj, ec, pruned, _ = _vs_oracle(at, 4, 1.1, params, phys)
    assert abs(res.forces[0, 0]) > 0.0  # shifted potential: zero energy, nonzero force at r_c
    np.testing.assert_allclose(res.forces, fref, rtol=1e-5, atol=1e-9)
    assert np.allclose(res.forces.sum(0), 0.0, atol=1e-9)
    beyond = _system([[1.0, 1.0, 1.0], [2.0 + 1e-9, 1.0, 1.0]], L, q=[0.4, -0.4])
    res2, fref2, _, _, pruned2, _ = _vs_oracle(beyond, 4, 1.1, params, phys)
    assert pruned2.masks.any()  # admitted (within r_list) ...
    assert np.array_equal(res2.forces, np.zeros((2, 3))) and res2.e_lj == 0.0 and res2.e_coulomb == 0.0  # ... no force
    assert np.array_equal(fref2, np.zeros((2, 3)))


def test_wrap_tiny_negative_and_box_length():
    nbx = _nbx()
    L = [3.0, 3.0, 3.0]
    s = _system([[-1e-17, 1.5, 1.5], [3.0, 1.0, 1.0], [1.5, -0.0, 3.0 - 1e-16], [2.9999999999999996, 2.0, 0.2]], L,
                q=[0.3, -0.3, 0.2, -0.2])
    params, phys = _cutoff_physics()
    res, fref, elj, ec, _, grid = _vs_oracle(s, 4, 1.1, params, phys)
    cp = grid.clustered_positions[~grid.fill_mask]
    assert np.all(cp >= 0.0) and np.all(cp < 3.0)  # wrapped into [0, L), never L itself
    np.testing.assert_allclose(res.forces, fref, rtol=1e-5, atol=1e-9)


def test_half_box_separation_and_newton():
    params, phys = _cutoff_physics(1.0)
    # exactly half a box apart along x (the minimum image picks the negative side)
    s = _system([[0.2, 1.0, 1.0], [1.2, 1.0, 1.0], [0.2, 1.9, 1.0]], [2.0, 2.5, 2.5], q=[0.5, -0.5, 0.1])
    res, fref, elj, ec, _, _ = _vs_oracle(s, 1, 1.0, params, phys)
    np.testing.assert_allclose(res.forces, fref, rtol=1e-5, atol=1e-9)
    # a random charged LJ fluid: the pair forces cancel (Newton's third law)
    rng = np.random.default_rng(3)
    L = np.array([3.2, 3.2, 3.2])
    g = (np.arange(8) + 0.5) * 0.4  # jittered 8^3 lattice: nearest neighbours >= 0.3 nm
    pos = np.stack(np.meshgrid(g, g, g, indexing="ij"), -1).reshape(-1, 3) + rng.uniform(-0.05, 0.05, (512, 3))
    n = pos.shape[0]
    q = rng.choice([-0.4, 0.4], n)
    res, fref, elj, ec, _, _ = _vs_oracle(_system(pos, L, q=q), 4, 1.1, params, phys)
    assert np.abs(res.forces.sum(0)).max() <= 1e-6 * np.abs(res.forces).max()
    assert np.sqrt(((res.forces - fref) ** 2).sum() / (fref ** 2).sum()) <= 1e-4
    assert abs(res.e_lj - elj) <= 1e-5 * abs(elj) and abs(res.e_coulomb - ec) <= 1e-5 * abs(ec)


def test_interaction_stats_two_isolated_particles():
    nbx = _nbx()
    # the reference's case: two particles 0.5 apart, m = 1, r_list = r_cut = 0.9
    s = _system([[1.0, 1.0, 1.0], [1.5, 1.0, 1.0]], [10.0, 10.0, 10.0])
    grid = nbx.build_cluster_grid(s, 1)
    st = nbx.interaction_stats(nbx.build_pair_list(grid, s.box, 0.9), grid, grid.clustered_positions, s.box, 0.9)
    assert (st.n_admitted, st.n_within_cutoff, st.ratio) == (1, 1, 1.0)
    # far apart: nothing admitted at m = 1; at m = 4 both share one cluster, whose
    # diagonal row admits the pair whatever its distance (pairlist.py:106-112)
    far = _system([[0.5, 0.5, 0.5], [3.0, 3.0, 3.0]], [6.0, 6.0, 6.0])
    for m, n_adm in ((1, 0), (4, 1)):
        grid = nbx.build_cluster_grid(far, m)
        plist = nbx.prune_pair_list(nbx.build_pair_list(grid, far.box, 1.1), grid.clustered_positions, far.box)
        st = nbx.interaction_stats(plist, grid, grid.clustered_positions, far.box, 1.0)
        assert (st.n_admitted, st.n_within_cutoff) == (n_adm, 0)
