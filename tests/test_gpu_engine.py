"""GPU engine pieces: parallel_forces, lifecycle / drift guard, integrator
(engine.py:294-580, oracle.py:88-123 of the reference)."""

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu


def _fluid(name="charged_fluid600"):
    import paper_1506_00716_b200 as nbx

    g = load_golden(name)
    n = g["positions"].shape[0]
    rng = np.random.default_rng(3)
    s = nbx.ParticleSystem(positions=g["positions"], velocities=rng.normal(scale=0.3, size=(n, 3)),
                           masses=g["masses"], charges=g["charges"], lj_type=g["lj_type"], box=nbx.SimBox(g["box"]))
    params = nbx.NonbondedParams(r_cut=float(g["r_cut"]), r_list=float(g["r_list"]), lj_table=g["lj_table"],
                                 shift_potential=bool(g["shift"]))
    return nbx, g, s, params


def test_parallel_forces_equals_api_and_is_worker_independent():
    nbx, g, s, params = _fluid()
    layout = nbx.KernelLayout(4, 4)
    st = nbx.init_state(s, params, layout)
    ref = nbx.compute_nonbonded_original(st.plist, st.grid, s.positions, s.charges, s.lj_type, params, s.box, layout)
    outs = [nbx.parallel_forces(st, params, layout, workers=w) for w in (1, 3, 8)]
    for o in outs:
        assert np.array_equal(o.forces, ref.forces)
        assert o.e_lj == ref.e_lj and o.e_coulomb == ref.e_coulomb
    with pytest.raises(nbx.ParameterError):
        nbx.parallel_forces(st, params, layout, workers=0)


def test_update_drift_matches_numpy_exactly():
    nbx, g, s, params = _fluid()
    rng = np.random.default_rng(9)
    tr = nbx.DriftTracker(reference_positions=nbx.wrap_position(s.positions, s.box))
    cur = s.positions + rng.normal(scale=0.05, size=s.positions.shape)
    cur[:10] += s.box.lengths  # periodic images must not count
    out = nbx.update_drift(tr, cur, s.box)
    disp = nbx.minimum_image(cur - tr.reference_positions, s.box)
    expect = float(np.sqrt(np.einsum("kd,kd->k", disp, disp).max()))   # oracle.py:119-121
    assert out.max_displacement == expect
    assert nbx.update_drift(out, tr.reference_positions, s.box).max_displacement == expect  # never decreases


def test_lifecycle_rebuilds_on_interval_and_guard():
    nbx, g, s, params = _fluid()
    layout = nbx.KernelLayout(4, 4)
    policy = nbx.ListPolicy(rebuild_interval=5)
    st = nbx.init_state(s, params, layout, policy=policy)
    st.step = 3
    assert not nbx.lifecycle_tick(st, params, policy)
    st.step = 5
    assert nbx.lifecycle_tick(st, params, policy) and st.n_rebuilds == 2
    st.drift = nbx.DriftTracker(reference_positions=st.drift.reference_positions,
                                max_displacement=0.6 * (params.r_list - params.r_cut))
    st.step = 6
    assert nbx.lifecycle_tick(st, params, policy) and st.n_drift_rebuilds == 1


def test_velocity_verlet_step_matches_reference_formula():
    nbx, g, s, params = _fluid()
    layout = nbx.KernelLayout(4, 4)
    policy = nbx.ListPolicy(rebuild_interval=10)
    st = nbx.init_state(s, params, layout, policy=policy)
    f0 = nbx.parallel_forces(st, params, layout)
    dt = 0.002
    x0, v0 = st.system.positions.copy(), st.system.velocities.copy()
    f1 = nbx.velocity_verlet_step(st, params, dt, f0, layout, policy=policy)
    inv_mass = (0.5 * dt) / s.masses[:, None]            # engine.py:556-563
    vh = v0 + f0.forces * inv_mass
    x1 = nbx.wrap_position(x0 + vh * dt, s.box)
    assert np.array_equal(st.system.positions, x1)
    v1 = vh + f1.forces * inv_mass
    assert np.array_equal(st.system.velocities, v1)
    assert st.step == 1
