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


def test_run_md_device_resident_matches_host_loop():
    """run_md (state on the GPU, engine.py:610-706) against the step-by-step
    host loop of velocity_verlet_step + lifecycle_tick on the same system."""
    nbx, g, s, params = _fluid("lj_fluid400")
    layout = nbx.KernelLayout(4, 4)
    policy = nbx.ListPolicy(rebuild_interval=7)
    dt, n_steps = 0.002, 30
    res = nbx.run_md(s, params, layout, dt, n_steps, policy=policy, report_interval=10)
    assert list(res.steps) == [0, 10, 20, 30]
    st = nbx.init_state(s, params, layout, policy=policy)
    f = nbx.parallel_forces(st, params, layout)
    ke, pe = [nbx.kinetic_energy(st.system)], [f.e_lj + f.e_coulomb]
    for k in range(1, n_steps + 1):
        f = nbx.velocity_verlet_step(st, params, dt, f, layout, policy=policy)
        if k % 10 == 0:
            ke.append(nbx.kinetic_energy(st.system))
            pe.append(f.e_lj + f.e_coulomb)
    assert res.state.step == st.step == n_steps
    assert res.state.n_rebuilds == st.n_rebuilds
    dx = nbx.minimum_image(res.state.system.positions - st.system.positions, s.box)
    assert np.abs(dx).max() < 1e-8
    assert np.allclose(res.state.system.velocities, st.system.velocities, rtol=1e-6, atol=1e-8)
    assert np.allclose(res.e_kinetic, ke, rtol=1e-9)
    assert np.allclose(res.e_potential, pe, rtol=1e-6)
    assert np.allclose(res.forces.forces, f.forces, rtol=1e-5, atol=1e-6)
    assert len(res.log_lines) == 2 + 4 + 1 and res.log_lines[-1].startswith("# energy drift")


def test_run_md_drift_guard_rebuilds():
    nbx, g, s, params = _fluid("lj_fluid400")
    layout = nbx.KernelLayout(4, 4)
    fast = nbx.ParticleSystem(positions=s.positions, velocities=s.velocities * 40.0, masses=s.masses,
                              charges=s.charges, lj_type=s.lj_type, box=s.box)
    res = nbx.run_md(fast, params, layout, 0.002, 20, policy=nbx.ListPolicy(rebuild_interval=1000),
                     report_interval=20)
    assert res.state.n_drift_rebuilds >= 1
    assert res.state.n_rebuilds == 1 + res.state.n_drift_rebuilds
    assert np.all(res.max_drift <= 0.5 * (params.r_list - params.r_cut) + 1e-12)
    with pytest.raises(nbx.ParameterError):
        nbx.run_md(s, params, layout, -1.0, 5)


def test_run_md_with_dynamic_pruning_matches_plain_run():
    """run_md with the inner force list and rolling prunes every 2 steps
    follows the same trajectory as without (same pairs within r_c; only the
    FP32 summation order may differ)."""
    nbx, g, s, params = _fluid("lj_fluid400")
    layout = nbx.KernelLayout(4, 4)
    r_inner = params.r_cut + 0.5 * (params.r_list - params.r_cut)
    a = nbx.run_md(s, params, layout, 0.002, 30, policy=nbx.ListPolicy(rebuild_interval=7), report_interval=10)
    b = nbx.run_md(s, params, layout, 0.002, 30, report_interval=10,
                   policy=nbx.ListPolicy(rebuild_interval=7, r_inner=r_inner, prune_interval=2))
    assert a.state.n_rebuilds == b.state.n_rebuilds
    dx = nbx.minimum_image(a.state.system.positions - b.state.system.positions, s.box)
    assert np.abs(dx).max() < 1e-7
    assert np.allclose(a.e_potential, b.e_potential, rtol=1e-6)
    assert np.allclose(a.forces.forces, b.forces.forces, rtol=1e-4, atol=1e-5)
    with pytest.raises(nbx.ParameterError):
        nbx.ListPolicy(r_inner=-0.1)
