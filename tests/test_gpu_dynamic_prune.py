"""Dynamic pruning (extension, BASELINE config 5): the inner force list.

`prune_pair_list(..., r_inner=R)` keeps the canonical r_list list unchanged
(the parity object) and gives the force kernel masks restricted to rows with
a pair within R at the build positions; the kernel uses them only while
2 d_max <= R - r_c (device-side check every call).  Forces must match the
full list and the oracle at the north_star tolerances, whether the inner
list is in use (small moves) or the kernel falls back (large moves)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

FORCE_RTOL = 1e-4
ENERGY_RTOL = 1e-5
R_INNER = 1.02


def _spc(n, m=4):
    import paper_1506_00716_b200 as nbx
    from paper_1506_00716_b200.systems import spc_water, tuned_occupancy

    s, table = spc_water(n, seed=2024)
    return nbx, s, table, tuned_occupancy(n, float(s.box.lengths[0]), m)


def rel_rms(f, ref):
    return float(np.sqrt(((f - ref) ** 2).sum() / (ref ** 2).sum()))


def rel(a, b):
    return abs(a - b) / abs(b)


def _params(nbx, table, elec):
    if elec == "ewald":
        return nbx.NonbondedParams(r_cut=1.0, r_list=1.1, lj_table=table, shift_potential=True, elec="ewald",
                                   ewald_beta=nbx.ewald_beta(1.0))
    return nbx.NonbondedParams(r_cut=1.0, r_list=1.1, lj_table=table, shift_potential=True)


@pytest.mark.parametrize("m", [4, 8])
@pytest.mark.parametrize("elec", ["ewald", "cutoff"])
def test_inner_list_keeps_rows_and_forces(m, elec):
    nbx, s, table, occ = _spc(24000, m)
    grid = nbx.build_cluster_grid(s, m, occ)
    built = nbx.build_pair_list(grid, s.box, 1.1)
    full = nbx.prune_pair_list(built, grid.clustered_positions_device, s.box)
    inner = nbx.prune_pair_list(built, grid.clustered_positions_device, s.box, r_inner=R_INNER)
    # the canonical list is the same object either way
    assert np.array_equal(inner.offsets, full.offsets)
    assert np.array_equal(inner.j_idx, full.j_idx)
    assert np.array_equal(inner.mask_bits, full.mask_bits)
    stats = nbx.interaction_stats(full, grid, grid.clustered_positions_device, s.box, 1.0)
    n_full, n_inner = full.force_pairs(), inner.force_pairs()
    assert n_full == stats.n_admitted == inner.force_pairs(inner=False)
    assert stats.n_within_cutoff <= n_inner < n_full
    params = _params(nbx, table, elec)
    layout = nbx.KernelLayout(m, 4)
    a = nbx.compute_nonbonded_original(full, grid, s.positions, s.charges, s.lj_type, params, s.box, layout)
    b = nbx.compute_nonbonded_original(inner, grid, s.positions, s.charges, s.lj_type, params, s.box, layout)
    # same pairs, another FP32 summation order
    assert rel_rms(b.forces, a.forces) <= 1e-6
    assert rel(b.e_lj, a.e_lj) <= 1e-7 and rel(b.e_coulomb, a.e_coulomb) <= 1e-7


@pytest.mark.parametrize("move", [0.004, 0.03])
def test_inner_list_under_motion_vs_oracle(move):
    """0.004 nm: 2 d_max < r_inner - r_c, the inner list is used; 0.03 nm:
    it is not (fallback to the full masks).  Both against the oracle on the
    moved positions with the same canonical list."""
    from oracle import forces as of
    from oracle import native, search

    nbx, s, table, occ = _spc(24000)
    L = s.box.lengths
    grid = nbx.build_cluster_grid(s, 4, occ)
    inner = nbx.prune_pair_list(nbx.build_pair_list(grid, s.box, 1.1), grid.clustered_positions_device, s.box,
                                r_inner=R_INNER)
    rng = np.random.default_rng(11)
    step = rng.normal(size=(s.n, 3))
    step *= move / np.linalg.norm(step, axis=1, keepdims=True)
    moved = s.positions + step
    params = _params(nbx, table, "ewald")
    res = nbx.compute_nonbonded_original(inner, grid, moved, s.charges, s.lj_type, params, s.box,
                                         nbx.KernelLayout(4, 4))
    og = search.build_grid(s.positions, L, 4, occ)
    ol = dict(m=4, offsets=inner.offsets, j_idx=inner.j_idx, masks=inner.masks, r_list=1.1)
    phys = of.Physics(r_cut=1.0, lj_table=table, shift_potential=True, elec="ewald",
                      ewald_beta=of.ewald_beta_for(1.0))
    fc, elj, ec = native.list_forces(ol, og, moved, s.charges, s.lj_type, L, phys)
    assert rel_rms(res.forces, search.scatter_to_original(og, fc)) <= FORCE_RTOL
    assert rel(res.e_lj, elj) <= ENERGY_RTOL and rel(res.e_coulomb, ec) <= ENERGY_RTOL


def test_inner_list_parameter_errors():
    nbx, s, table, occ = _spc(3000)
    grid = nbx.build_cluster_grid(s, 4, occ)
    built = nbx.build_pair_list(grid, s.box, 1.1)
    with pytest.raises(nbx.ParameterError):
        nbx.prune_pair_list(built, grid.clustered_positions_device, s.box, r_inner=1.2)
    with pytest.raises(nbx.ParameterError):
        nbx.prune_pair_list(built, grid.clustered_positions_device, s.box, r_inner=-0.5)
    # the d_max guard is measured against the build positions: other prune
    # positions cannot carry an inner list
    other = np.array(grid.clustered_positions) + 0.001
    with pytest.raises(nbx.ParameterError):
        nbx.prune_pair_list(built, other, s.box, r_inner=R_INNER)


def test_rolling_prune_vs_oracle():
    """Rolling prune (NBX_FORCE_REPRUNE): after atoms moved past the inner
    list's margin (fallback pass), the inner list is redone at those
    positions; a later small move uses it, a large one falls back again --
    every pass against the oracle on the same canonical list."""
    import torch

    from oracle import forces as of
    from oracle import native, search

    nbx, s, table, occ = _spc(24000)
    L = s.box.lengths
    grid = nbx.build_cluster_grid(s, 4, occ)
    pl = nbx.prune_pair_list(nbx.build_pair_list(grid, s.box, 1.1), grid.clustered_positions_device, s.box,
                             r_inner=R_INNER)
    n_full = pl.force_pairs(inner=False)
    params = _params(nbx, table, "ewald")
    og = search.build_grid(s.positions, L, 4, occ)
    ol = dict(m=4, offsets=pl.offsets, j_idx=pl.j_idx, masks=pl.masks, r_list=1.1)
    phys = of.Physics(r_cut=1.0, lj_table=table, shift_potential=True, elec="ewald",
                      ewald_beta=of.ewald_beta_for(1.0))
    dev = torch.device("cuda", 0)
    q = torch.as_tensor(np.array(s.charges), device=dev)
    t = torch.as_tensor(np.array(s.lj_type), device=dev)
    rng = np.random.default_rng(3)

    def moved(base, d):
        st = rng.normal(size=(s.n, 3))
        return base + st * (d / np.linalg.norm(st, axis=1, keepdims=True))

    def check(p, reprune=False):
        f, e, _ = nbx.compute_nonbonded_device(pl, grid, torch.as_tensor(p, device=dev), q, t, params, s.box,
                                               reprune=reprune)
        fc, elj, ec = native.list_forces(ol, og, p, s.charges, s.lj_type, L, phys)
        eh = e.cpu().numpy()
        assert rel_rms(f.cpu().numpy(), search.scatter_to_original(og, fc)) <= FORCE_RTOL
        assert rel(eh[0], elj) <= ENERGY_RTOL and rel(eh[1], ec) <= ENERGY_RTOL

    p1 = moved(s.positions, 0.03)
    check(p1, reprune=True)            # fallback pass, then the inner list is redone at p1
    assert pl.force_pairs(inner=True) < n_full
    check(moved(p1, 0.004))            # inner list (from p1) in use
    p3 = moved(p1, 0.004)
    check(p3, reprune=True)            # in use, and redone at p3
    check(moved(p3, 0.03))             # fallback from the p3 prune
