"""Rigid-water oracle (CPU, test infrastructure): SETTLE against iterated
SHAKE, RATTLE's velocity stage, and the exclusion restatement."""

import numpy as np

from oracle import native, search
from oracle.constraints import rattle_velocities, settle_positions, shake_positions
from oracle.geometry import min_image
from paper_1506_00716_b200.systems import spc_water, tuned_occupancy

D_OH = 0.1
D_HH = 2.0 * 0.1 * np.sin(np.deg2rad(109.47) / 2.0)


def _bond(x, i, j, L):
    x = x.reshape(-1, 3, 3)
    return np.linalg.norm(min_image(x[:, j] - x[:, i], L), axis=1)


def _drifted(n=3000, seed=1, dt=0.002):
    s, _ = spc_water(n, seed=2024)
    L = np.asarray(s.box.lengths)
    m = np.array(s.masses)
    rng = np.random.default_rng(seed)
    v = rng.normal(size=(n, 3)) * np.sqrt(2.494 / m)[:, None]
    return s, L, m, v, np.array(s.positions), np.array(s.positions) + v * dt


def test_settle_matches_shake_and_holds_geometry():
    s, L, m, v, x0, x1 = _drifted()
    xs, ds = settle_positions(x0, x1, m, L, D_OH, D_HH)
    xk, dk = shake_positions(x0, x1, m, L, D_OH, D_HH)
    assert np.abs(ds - dk).max() < 1e-13
    for i, j, d in ((0, 1, D_OH), (0, 2, D_OH), (1, 2, D_HH)):
        assert np.abs(_bond(xs, i, j, L) - d).max() < 1e-13
    # constraint forces are internal: no momentum change per molecule
    assert np.abs((m[:, None] * ds).reshape(-1, 3, 3).sum(axis=1)).max() < 1e-14


def test_rattle_removes_bond_velocities_only():
    s, L, m, v, x0, _ = _drifted()
    vr = rattle_velocities(x0, v, m, L)
    xr, vv = x0.reshape(-1, 3, 3), vr.reshape(-1, 3, 3)
    for i, j in ((0, 1), (0, 2), (1, 2)):
        assert np.abs(np.einsum("kd,kd->k", min_image(xr[:, j] - xr[:, i], L), vv[:, j] - vv[:, i])).max() < 1e-12
    assert np.abs((m[:, None] * (vr - v)).reshape(-1, 3, 3).sum(axis=1)).max() < 1e-12
    # idempotent
    assert np.abs(rattle_velocities(x0, vr, m, L) - vr).max() < 1e-12


def test_exclusion_restatement_removes_only_intramolecular_pairs():
    s, _ = spc_water(3000, seed=2024)
    L = np.asarray(s.box.lengths)
    g = search.build_grid(s.positions, L, 4, tuned_occupancy(3000, float(L[0]), 4))
    lst = native.search_list(g, L, 1.1)
    ex = search.exclude_molecules(lst, g, np.arange(3000) // 3)
    removed = int(lst["masks"].sum() - ex["masks"].sum())
    # every molecule has its 3 intramolecular pairs within r_list: each is
    # admitted exactly once in the half list
    assert removed == 3 * 1000
    assert np.all(ex["masks"] <= lst["masks"])
