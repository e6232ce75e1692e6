"""Rigid SPC water on the GPU (extension): molecule exclusions
in the lists, SETTLE / RATTLE kernels against the oracle restatements
(oracle/constraints.py, itself pinned to iterated SHAKE), and a stable
rigid-water run_md."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

FORCE_RTOL = 1e-4
ENERGY_RTOL = 1e-5


def _spc(n):
    import paper_1506_00716_b200 as nbx
    from paper_1506_00716_b200.systems import spc_water, tuned_occupancy

    s, table = spc_water(n, seed=2024)
    return nbx, s, table, tuned_occupancy(n, float(s.box.lengths[0]), 4)


def rel_rms(f, ref):
    return float(np.sqrt(((f - ref) ** 2).sum() / (ref ** 2).sum()))


def test_exclusions_lists_and_forces_vs_oracle():
    from oracle import forces as of
    from oracle import native, search

    nbx, s, table, occ = _spc(3000)
    L = s.box.lengths
    mol = np.arange(s.n) // 3
    grid = nbx.build_cluster_grid(s, 4, occ)
    built = nbx.build_pair_list(grid, s.box, 1.1, molecules=mol)
    pruned = nbx.prune_pair_list(built, grid.clustered_positions, s.box)
    og = search.build_grid(s.positions, L, 4, occ)
    ob = search.exclude_molecules(native.search_list(og, L, 1.1), og, mol)
    op = native.prune_list(ob, og["clustered_positions"], L)
    assert np.array_equal(built.mask_bits, search.pack_masks(ob["masks"]))
    assert np.array_equal(pruned.offsets, op["offsets"]) and np.array_equal(pruned.j_idx, op["j_idx"])
    assert np.array_equal(pruned.mask_bits, search.pack_masks(op["masks"]))
    # the exclusion count (3 intramolecular pairs per molecule)
    again = nbx.build_pair_list(grid, s.box, 1.1)
    assert nbx.exclude_molecules(again, mol, count=True) == 3 * (s.n // 3)
    params = nbx.NonbondedParams(r_cut=1.0, r_list=1.1, lj_table=table, elec="reaction_field", epsilon_rf=0.0)
    phys = of.Physics(r_cut=1.0, lj_table=table, elec="reaction_field", epsilon_rf=0.0)
    res = nbx.compute_nonbonded_original(pruned, grid, s.positions, s.charges, s.lj_type, params, s.box,
                                         nbx.KernelLayout(4, 4))
    fb, elj, ec, (alj, ac) = of.brute_force(s.positions, s.charges, s.lj_type, L, phys, molecules=mol,
                                            abs_sums=True)
    assert rel_rms(res.forces, fb) <= FORCE_RTOL
    # without the intramolecular terms the Coulomb total (~ -330) is a
    # cancellation of pair energies ~3 orders larger: the energy bar is taken
    # relative to the summed magnitudes (FP32 pair terms, FP64 sums)
    assert abs(res.e_lj - elj) <= ENERGY_RTOL * alj
    assert abs(res.e_coulomb - ec) <= ENERGY_RTOL * ac, (res.e_coulomb, ec, ac)


def test_settle_and_rattle_kernels_vs_oracle():
    import torch

    from oracle.constraints import rattle_velocities, settle_positions
    from paper_1506_00716_b200.engine import settle_device

    nbx, s, table, occ = _spc(24000)
    L = np.asarray(s.box.lengths)
    m = np.array(s.masses)
    rng = np.random.default_rng(3)
    v = rng.normal(size=(s.n, 3)) * np.sqrt(2.494 / m)[:, None]
    dt = 0.002
    x0 = np.array(s.positions)
    x1 = np.mod(x0 + v * dt, L)  # drifted and wrapped per atom
    water = nbx.RigidWater()
    xs_ref, disp = settle_positions(x0, x1, m, L, water.d_oh, water.d_hh)
    xd = torch.tensor(x1, device="cuda")
    vd = torch.tensor(v, device="cuda")
    settle_device(torch.tensor(x0, device="cuda"), xd, vd, water, m[0], m[1], dt, s.box)
    dx = xd.cpu().numpy() - xs_ref
    dx -= L * np.round(dx / L)
    assert np.abs(dx).max() < 1e-11
    assert np.abs(vd.cpu().numpy() - (v + disp / dt)).max() < 1e-8
    vr_ref = rattle_velocities(xs_ref, v, m, L)
    vd = torch.tensor(v, device="cuda")
    settle_device(None, torch.tensor(xs_ref, device="cuda"), vd, water, m[0], m[1], dt, s.box, velocities_only=True)
    assert np.abs(vd.cpu().numpy() - vr_ref).max() < 1e-10


def test_rigid_water_md_is_stable():
    """24k SPC water, reaction field (eps_rf = inf), dt = 2 fs, 400 steps
    with molecule exclusions + SETTLE: bonds stay rigid to rounding, the
    temperature stays near its start, total energy drifts little."""
    from oracle.geometry import min_image

    nbx, _, table, occ = _spc(24000)
    from paper_1506_00716_b200.systems import spc_water

    s, table = spc_water(24000, seed=2024, temperature=300.0)
    params = nbx.NonbondedParams(r_cut=1.0, r_list=1.1, lj_table=table, elec="reaction_field", epsilon_rf=0.0)
    water = nbx.RigidWater()
    res = nbx.run_md(s, params, nbx.KernelLayout(4, 4), 0.002, 400, report_interval=50,
                     target_occupancy=occ, constraints=water)
    x = res.state.system.positions.reshape(-1, 3, 3)
    L = np.asarray(s.box.lengths)
    for i, j, d in ((0, 1, water.d_oh), (0, 2, water.d_oh), (1, 2, water.d_hh)):
        assert np.abs(np.linalg.norm(min_image(x[:, j] - x[:, i], L), axis=1) - d).max() < 1e-9
    assert np.all(np.isfinite(res.e_total))
    # the generated lattice relaxes during the first ~50 steps (its potential
    # energy turns into heat, NVE); after that the run must conserve energy:
    # total-energy excursion below 2 % of the kinetic energy, temperature flat
    e = res.e_total[2:]
    ke = res.e_kinetic[2:]
    assert np.abs(e - e[0]).max() < 0.02 * ke.mean(), (res.e_total, res.e_kinetic)
    t = res.temperature[2:]
    assert np.abs(t - t.mean()).max() < 0.05 * t.mean(), res.temperature


def test_fused_constrained_integration_is_bit_identical(monkeypatch):
    """nbx_vv_constrained (half kick + drift + SETTLE, half kick + RATTLE in
    one kernel each) reproduces the separate kernels bit for bit."""
    nbx, _, table, occ = _spc(3000)
    from paper_1506_00716_b200.systems import spc_water

    s, table = spc_water(3000, seed=7, temperature=300.0)
    params = nbx.NonbondedParams(r_cut=1.0, r_list=1.1, lj_table=table, elec="reaction_field", epsilon_rf=0.0)
    water = nbx.RigidWater()
    runs = []
    for fused in ("1", "0"):
        monkeypatch.setenv("NBX_MD_FUSED", fused)
        runs.append(nbx.run_md(s, params, nbx.KernelLayout(4, 4), 0.002, 60, report_interval=10,
                               target_occupancy=occ, constraints=water))
    a, b = runs
    assert np.array_equal(a.state.system.positions, b.state.system.positions)
    assert np.array_equal(a.state.system.velocities, b.state.system.velocities)
    assert np.array_equal(a.e_total, b.e_total)
