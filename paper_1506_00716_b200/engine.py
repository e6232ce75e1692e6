"""List lifecycle, drift guard and the force pass of an MD step -- GPU-backed
drop-in for the hot-path part of clustermd.engine.

Mirrors /root/reference/pkg/src/clustermd/engine.py: ``ListPolicy``,
``MDState``, ``init_state`` (:337-384), ``lifecycle_tick`` (:387-406),
``parallel_forces`` (:462-521) and ``velocity_verlet_step`` (:543-580);
``DriftTracker`` / ``update_drift`` mirror oracle.py:88-123.

The force pass is one GPU launch sequence whatever ``workers`` is: the
reference's per-worker buffers and fixed-order reduction (engine.py:485-514)
are replaced by the library's deterministic reduction, so results are
bit-identical across reruns *and* across worker counts.
"""

from __future__ import annotations

import os
import time
from contextlib import contextmanager
from dataclasses import dataclass, field, replace

import numpy as np
import torch

from . import _device as dev
from . import _lib
from .gridder import ClusterGrid, build_cluster_grid
from .kernels import KernelLayout, compute_nonbonded_original
from .model import (BOLTZMANN_KJ_MOL_K, ForcesEnergies, NonbondedParams, ParameterError, ParticleSystem,
                    SimBox, wrap_position)
from .pairlist import ClusterPairList, Molecules, build_pair_list, list_step, prune_pair_list


# ---------------------------------------------------------------- timing (host bookkeeping)
class TimingError(RuntimeError):
    """Improper section nesting (engine.py:35-36)."""


class TimingReport:
    """Named nested wall-time sections (engine.py:45-121), kept so callers of
    the reference API can pass a timer; device work is timed with CUDA events
    elsewhere (bench.py, tools/step_breakdown.py)."""

    def __init__(self, debug: bool = False):
        self.debug = debug
        self.sections: dict = {}
        self.parent: dict = {}
        self._stack: list = []

    @contextmanager
    def section(self, name: str):
        if name in self._stack:
            if self.debug:
                raise TimingError(f"section {name!r} re-entered while active")
            yield self
            return
        parent = self._stack[-1] if self._stack else None
        if self.parent.get(name, parent) != parent and self.debug:
            raise TimingError(f"section {name!r} opened under {parent!r}")
        self.parent.setdefault(name, parent)
        entry = self.sections.setdefault(name, [0, 0.0])
        self._stack.append(name)
        t0 = time.perf_counter()
        try:
            yield self
        finally:
            entry[1] += time.perf_counter() - t0
            entry[0] += 1
            self._stack.pop()

    def total(self, name: str) -> float:
        return self.sections[name][1]


@contextmanager
def _maybe(timer, name):
    if timer is None:
        yield
    else:
        with timer.section(name):
            yield


# ---------------------------------------------------------------- drift guard
@dataclass(frozen=True)
class DriftTracker:
    """Largest minimum-image displacement since the reference snapshot (oracle.py:88-103)."""

    reference_positions: np.ndarray
    max_displacement: float = 0.0

    def __post_init__(self):
        ref = np.array(self.reference_positions, dtype=np.float64, copy=True).reshape(-1, 3)
        ref.setflags(write=False)
        object.__setattr__(self, "reference_positions", ref)


_disp_scratch: dict = {}  # device index -> 16-byte zeroed scratch of nbx_max_displacement_ex


def max_displacement_device(ref: torch.Tensor, cur: torch.Tensor, box: SimBox) -> torch.Tensor:
    """Device scalar: max_i |minimum_image(cur_i - ref_i)| (no host sync;
    one kernel launch)."""
    out = torch.empty(1, dtype=torch.float64, device=cur.device)
    scratch = _disp_scratch.get(cur.device.index)
    if scratch is None:
        scratch = _disp_scratch[cur.device.index] = torch.zeros(2, dtype=torch.int64, device=cur.device)
    L = _lib.box3(box.lengths)
    _lib.check(_lib.load().nbx_max_displacement_ex(_lib.ptr(ref), _lib.ptr(cur), int(cur.shape[0]), _lib.ptr(L),
                                                   _lib.ptr(scratch), _lib.ptr(out), 1, dev.stream()),
               "max_displacement")
    return out


def update_drift(tracker: DriftTracker, current_positions, box: SimBox) -> DriftTracker:
    """Fold the current positions into the tracked maximum (oracle.py:106-123),
    evaluated on the GPU (bit-identical max)."""
    cur = np.asarray(current_positions, dtype=np.float64).reshape(-1, 3)
    if cur.shape != tracker.reference_positions.shape:
        raise ParameterError(f"positions shape {cur.shape} does not match reference "
                             f"{tracker.reference_positions.shape}")
    if cur.shape[0] == 0:
        return tracker
    d = max_displacement_device(dev.to_device(tracker.reference_positions, torch.float64),
                                dev.to_device(cur, torch.float64), box)
    largest = float(d.item())
    return DriftTracker(reference_positions=tracker.reference_positions,
                        max_displacement=max(tracker.max_displacement, largest))


# ---------------------------------------------------------------- lifecycle
@dataclass
class ListPolicy:
    """engine.py:266-277."""

    rebuild_interval: int = 10
    prune_on_build: bool = True
    # dynamic pruning (extension, run_md): inner force list at r_inner built
    # with each pruned list, redone at the current positions every
    # prune_interval steps (rolling prune); 0 = off
    r_inner: float = 0.0
    prune_interval: int = 0

    def __post_init__(self):
        if self.rebuild_interval < 1:
            raise ParameterError(f"rebuild_interval must be >= 1, got {self.rebuild_interval}")
        if self.r_inner < 0.0 or self.prune_interval < 0:
            raise ParameterError(f"r_inner and prune_interval must be >= 0, got {self.r_inner}, "
                                 f"{self.prune_interval}")


@dataclass(frozen=True)
class RigidWater:
    """Rigid 3-site water (extension: the reference has neither
    exclusions nor constraints, so its SPC water cannot be integrated, SURVEY
    0.3).  Molecules are atoms (3k, 3k+1, 3k+2) = (O, H, H) -- the order of
    systems.spc_water -- held rigid by SETTLE (positions) and RATTLE's
    velocity stage (nbx_settle), with every intramolecular pair excluded
    from the non-bonded list (pairlist.exclude_molecules).  Defaults: SPC
    geometry (O-H 0.1 nm, H-O-H 109.47 deg)."""

    d_oh: float = 0.1
    d_hh: float = 2.0 * 0.1 * float(np.sin(np.deg2rad(109.47) / 2.0))

    def molecules(self, n: int) -> np.ndarray:
        return np.arange(n, dtype=np.int64) // 3

    def check(self, system: ParticleSystem) -> tuple[float, float]:
        """(m_O, m_H) after validating the layout of ``system``."""
        n = system.n
        if n % 3:
            raise ParameterError(f"rigid water needs 3 atoms per molecule, got n={n}")
        if not (0.0 < 0.5 * self.d_hh < self.d_oh):
            raise ParameterError(f"invalid water geometry d_oh={self.d_oh}, d_hh={self.d_hh}")
        mm = system.masses.reshape(-1, 3)
        if n and not (np.all(mm[:, 0] == mm[0, 0]) and np.all(mm[:, 1:] == mm[0, 1])):
            raise ParameterError("rigid water needs identical (O, H, H) masses in every molecule")
        return (float(mm[0, 0]), float(mm[0, 1])) if n else (1.0, 1.0)

    def dof(self, n: int) -> int:
        return max(6 * (n // 3) - 3, 1)


def vv_constrained_device(x, v, f, m, water: RigidWater, m_o: float, m_h: float, dt: float, box: SimBox,
                          phase: int) -> None:
    """Rigid water: one velocity-Verlet half fused with its constraint
    (phase 0: half kick + drift + SETTLE; phase 1: half kick + RATTLE),
    nbx_vv_constrained -- bit-identical to vv_half_kick_device followed by
    settle_device."""
    L = _lib.box3(box.lengths)
    _lib.check(_lib.load().nbx_vv_constrained(_lib.ptr(x), _lib.ptr(v), _lib.ptr(f), _lib.ptr(m), int(x.shape[0]) // 3,
                                              float(m_o), float(m_h), float(water.d_oh), float(water.d_hh),
                                              float(dt), int(phase), _lib.ptr(L), dev.stream()), "vv_constrained")


def settle_device(x_old, x, v, water: RigidWater, m_o: float, m_h: float, dt: float, box: SimBox,
                  velocities_only: bool = False) -> None:
    """SETTLE of the drifted positions x (with v += displacement / dt), or --
    velocities_only -- RATTLE's velocity projection (device, in place)."""
    L = _lib.box3(box.lengths)
    _lib.check(_lib.load().nbx_settle(_lib.ptr(x_old) if x_old is not None else None, _lib.ptr(x), _lib.ptr(v),
                                      int(x.shape[0]) // 3, float(m_o), float(m_h), float(water.d_oh),
                                      float(water.d_hh), float(dt), 1 if velocities_only else 0, _lib.ptr(L),
                                      dev.stream()), "settle")


@dataclass
class MDState:
    """engine.py:280-291 (+ optional grid occupancy for the compact-cluster grid)."""

    system: ParticleSystem
    step: int
    grid: ClusterGrid
    plist: ClusterPairList
    drift: DriftTracker
    n_rebuilds: int = 0
    n_drift_rebuilds: int = 0
    slabs: object | None = None  # always None: see init_state
    target_occupancy: float | None = None


def _build(system, params, m, supercluster_size, n_lane, step, policy, occupancy, molecules=None):
    """engine.py:301-314: grid, list, and the prune of a reused list."""
    grid = build_cluster_grid(system, m, occupancy)
    plist = build_pair_list(grid, system.box, params.r_list, supercluster_size=supercluster_size,
                            n_lane=n_lane, build_step=step, molecules=molecules)
    if policy.prune_on_build and policy.rebuild_interval > 1:
        # the same inner list (dynamic pruning) as run_md's rebuilds
        plist = prune_pair_list(plist, grid.clustered_positions_device, system.box,
                                r_inner=min(policy.r_inner, params.r_list))
    return grid, plist


def _rebuild(state: MDState, params: NonbondedParams, policy: ListPolicy, timer) -> None:
    """engine.py:294-334."""
    with _maybe(timer, "grid_build"), _maybe(timer, "list_build"):
        state.grid, state.plist = _build(state.system, params, state.grid.m, state.plist.supercluster_size,
                                         state.plist.n_lane, state.step, policy, state.target_occupancy)
    state.drift = DriftTracker(reference_positions=wrap_position(state.system.positions, state.system.box))
    state.n_rebuilds += 1


def init_state(system: ParticleSystem, params: NonbondedParams, layout: KernelLayout, *,
               supercluster_size: int = 1, policy: ListPolicy | None = None, n_slabs: int = 0,
               slab_min_width: float | None = None, timer=None, target_occupancy: float | None = None,
               molecules=None) -> MDState:
    """Initial grid, list (pruned when reused) and optional slabs (engine.py:337-384)."""
    if params.r_list < params.r_cut:
        raise ParameterError(f"r_list={params.r_list} must be >= r_cut={params.r_cut}")
    policy = policy or ListPolicy()
    grid, plist = _build(system, params, layout.m, supercluster_size, layout.n_lane, 0, policy, target_occupancy,
                         molecules)
    state = MDState(system=system, step=0, grid=grid, plist=plist,
                    drift=DriftTracker(reference_positions=wrap_position(system.positions, system.box)),
                    n_rebuilds=1, target_occupancy=target_occupancy)
    if n_slabs < 0:
        raise ParameterError(f"n_slabs must be >= 0, got {n_slabs}")
    # n_slabs / slab_min_width are accepted for signature compatibility: one
    # GPU pass needs no work slabs, and the multi-GPU decomposition is
    # dd.SlabDecomposition (with its own cost-quantile rebalancing)
    return state


def lifecycle_tick(state: MDState, params: NonbondedParams, policy: ListPolicy, timer=None) -> bool:
    """Rebuild when the interval is due or 2 d_max > r_list - r_c (engine.py:387-406)."""
    interval_due = state.step - state.plist.build_step >= policy.rebuild_interval
    guard_due = 2.0 * state.drift.max_displacement > params.r_list - params.r_cut
    if not (interval_due or guard_due):
        return False
    if guard_due and not interval_due:
        state.n_drift_rebuilds += 1
    _rebuild(state, params, policy, timer)
    return True


def parallel_forces(state: MDState, params: NonbondedParams, layout: KernelLayout, workers: int = 1,
                    timer=None) -> ForcesEnergies:
    """Force pass over the current list, original order (engine.py:462-521).

    ``workers`` is validated for API compatibility; the GPU pass is one
    deterministic launch sequence, so results do not depend on it."""
    if workers < 1:
        raise ParameterError(f"workers must be >= 1, got {workers}")
    s = state.system
    res = compute_nonbonded_original(state.plist, state.grid, s.positions, s.charges, s.lj_type, params, s.box,
                                     layout)
    return res


# ---------------------------------------------------------------- integrator (device arithmetic)
def kinetic_energy(system: ParticleSystem) -> float:
    return 0.5 * float(np.einsum("k,kd,kd->", system.masses, system.velocities, system.velocities))


def temperature(system: ParticleSystem) -> float:
    n = system.n
    if n == 0:
        return 0.0
    dof = 3 * n - 3 if n > 1 else 3
    return 2.0 * kinetic_energy(system) / (dof * BOLTZMANN_KJ_MOL_K)


def total_momentum(system: ParticleSystem) -> np.ndarray:
    return np.einsum("k,kd->d", system.masses, system.velocities)


def vv_half_kick_device(x, v, f, mass, dt: float, box: SimBox, move: bool) -> None:
    """v += f (0.5 dt / m), then x = wrap(x + v dt) when ``move`` (device, in place)."""
    L = _lib.box3(box.lengths)
    _lib.check(_lib.load().nbx_vv_update(_lib.ptr(x), _lib.ptr(v), _lib.ptr(f), _lib.ptr(mass), int(x.shape[0]),
                                         float(dt), int(bool(move)), _lib.ptr(L), dev.stream()), "vv_update")


def velocity_verlet_step(state: MDState, params: NonbondedParams, dt: float, forces_in: ForcesEnergies,
                         layout: KernelLayout, *, policy: ListPolicy | None = None, workers: int = 1,
                         timer=None) -> ForcesEnergies:
    """One NVE step (engine.py:543-580); the half kicks, drift and wrap run on
    the GPU with the reference's FP64 operation order."""
    policy = policy or ListPolicy()
    s = state.system
    with _maybe(timer, "integrate"):
        x = dev.to_device(s.positions, torch.float64)
        v = dev.to_device(s.velocities, torch.float64)
        m = dev.to_device(s.masses, torch.float64)
        vv_half_kick_device(x, v, dev.to_device(forces_in.forces, torch.float64), m, dt, s.box, move=True)
        positions = x.cpu().numpy()
        state.system = replace(s, positions=positions, velocities=v.cpu().numpy())
        state.step += 1
        state.drift = update_drift(state.drift, positions, s.box)
    with _maybe(timer, "lifecycle"):
        lifecycle_tick(state, params, policy, timer)
    with _maybe(timer, "forces"):
        out = parallel_forces(state, params, layout, workers, timer)
    with _maybe(timer, "integrate"):
        v = dev.to_device(state.system.velocities, torch.float64)
        x = dev.to_device(state.system.positions, torch.float64)
        vv_half_kick_device(x, v, dev.to_device(out.forces, torch.float64), m, dt, s.box, move=False)
        state.system = replace(state.system, velocities=v.cpu().numpy())
    return out


@dataclass
class RunResult:
    """engine.py:583-607: final state plus the per-interval series of one run."""

    state: MDState
    forces: ForcesEnergies
    steps: np.ndarray
    e_kinetic: np.ndarray
    e_potential: np.ndarray
    temperature: np.ndarray = field(default_factory=lambda: np.zeros(0))
    max_drift: np.ndarray = field(default_factory=lambda: np.zeros(0))
    timing: TimingReport = field(default_factory=TimingReport)
    wall_seconds: float = 0.0
    log_lines: list = field(default_factory=list)

    @property
    def e_total(self) -> np.ndarray:
        return self.e_kinetic + self.e_potential

    def energy_drift(self) -> tuple[float, float]:
        """(max absolute, max relative) total-energy deviation from step 0."""
        e = self.e_total
        d = float(np.abs(e - e[0]).max()) if e.shape[0] else 0.0
        scale = abs(float(e[0])) if e.shape[0] else 0.0
        return d, d / scale if scale > 0 else d


def run_md(system: ParticleSystem, params: NonbondedParams, layout: KernelLayout, dt: float, n_steps: int, *,
           supercluster_size: int = 1, policy: ListPolicy | None = None, workers: int = 1, n_slabs: int = 0,
           slab_min_width: float | None = None, report_interval: int = 100, timer: TimingReport | None = None,
           target_occupancy: float | None = None, constraints: RigidWater | None = None) -> RunResult:
    """NVE velocity-Verlet run with the state resident on the GPU
    (engine.py:610-706 semantics).

    Positions, velocities and forces never leave the device between reports:
    per step one fused half-kick + drift + wrap kernel (``nbx_vv_update``),
    the drift guard as a device max-reduction (``nbx_max_displacement``; its
    single scalar is the only per-step host read), the list lifecycle
    (rebuild on interval or 2 d_max > r_list - r_c, grid built from the
    device positions), the force pass (energies only on report steps, like
    nstcalcenergy) and the second half kick.  Reports read back the
    energies and the kinetic energy; a singular pair raises at the next
    report (SingularityError, original indices) as the reference does at
    the failing step.

    ``constraints`` (extension): a RigidWater spec makes the run rigid-water
    MD -- intramolecular pairs excluded from every list, SETTLE after the
    drift, RATTLE's velocity stage after the second kick, temperature over
    6 n_mol - 3 degrees of freedom."""
    if dt <= 0.0:
        raise ParameterError(f"dt must be positive, got {dt}")
    if n_steps < 0:
        raise ParameterError(f"n_steps must be >= 0, got {n_steps}")
    if workers < 1:
        raise ParameterError(f"workers must be >= 1, got {workers}")
    if report_interval < 1:
        raise ParameterError(f"report_interval must be >= 1, got {report_interval}")
    from .kernels import _raise_if_singular, compute_nonbonded_device

    policy = policy or ListPolicy()
    timer = timer or TimingReport()
    wall0 = time.perf_counter()
    d = dev.require_cuda()
    box = system.box
    buffer = params.r_list - params.r_cut
    mol = None
    if constraints is not None:
        m_o, m_h = constraints.check(system)
        mol = Molecules(constraints.molecules(system.n))  # device topology, built once
    with timer.section("setup"):
        state = init_state(system, params, layout, supercluster_size=supercluster_size, policy=policy,
                           n_slabs=n_slabs, slab_min_width=slab_min_width, target_occupancy=target_occupancy,
                           molecules=mol)
        x = dev.to_device(system.positions, torch.float64).clone()
        v = dev.to_device(system.velocities, torch.float64).clone()
        # rigid water: each velocity-Verlet half fused with its constraint
        # (bit-identical; NBX_MD_FUSED=0 runs the separate kernels)
        fused = constraints is not None and os.environ.get("NBX_MD_FUSED", "1") != "0"
        x_old = torch.empty_like(x) if constraints is not None and not fused else None
        if constraints is not None:  # start from velocities that keep the bonds rigid
            settle_device(None, x, v, constraints, m_o, m_h, dt, box, velocities_only=True)
        m = dev.to_device(system.masses, torch.float64)
        q = dev.to_device(system.charges, torch.float64)
        ty = dev.to_device(system.lj_type, torch.int64)
        ref = dev.to_device(state.drift.reference_positions, torch.float64).clone()
        f = torch.empty_like(x)
        e = torch.zeros(2, dtype=torch.float64, device=d)
        bad = torch.empty(2, dtype=torch.int64, device=d)
        d_max = d_last = 0.0
        d_pin = torch.zeros(1, dtype=torch.float64).pin_memory()
        d_ev = torch.cuda.Event()

        def force_pass(energy: bool):
            age = state.step - state.plist.build_step
            rp = policy.r_inner > 0.0 and policy.prune_interval > 0 and age > 0 and age % policy.prune_interval == 0
            compute_nonbonded_device(state.plist, state.grid, x, q, ty, params, box, energy=energy, out=f,
                                     e_out=e, bad=bad, reprune=rp)

        force_pass(True)

    steps, e_kin, e_pot, temps, drifts = [], [], [], [], []
    log = ["# clustermd run log", "# step e_kinetic e_potential e_total temperature_K max_drift_nm"]
    dof = 3 * system.n - 3 if system.n > 1 else 3
    if constraints is not None:
        dof = constraints.dof(system.n)

    def record():
        # one device->host read: energies, kinetic energy, singular-pair key
        vals = torch.cat([e, torch.einsum("k,kd,kd->", m, v, v).reshape(1), bad.to(torch.float64)]).cpu().numpy()
        bad_h = vals[3:5].astype(np.int64)
        _raise_if_singular(state.plist, state.grid, x, bad_h, params, box)
        ke = 0.5 * float(vals[2])
        pe = float(vals[0] + vals[1])
        steps.append(state.step)
        e_kin.append(ke)
        e_pot.append(pe)
        temps.append(2.0 * ke / (dof * BOLTZMANN_KJ_MOL_K) if system.n else 0.0)
        drifts.append(d_max)
        log.append(f"{state.step} {ke:.10e} {pe:.10e} {ke + pe:.10e} {temps[-1]:.6f} {d_max:.6e}")

    record()
    for _ in range(n_steps):
        with timer.section("step"):
            with timer.section("integrate"):
                if fused:  # half kick + drift + SETTLE in one kernel
                    vv_constrained_device(x, v, f, m, constraints, m_o, m_h, dt, box, phase=0)
                else:
                    if constraints is not None:
                        x_old.copy_(x)
                    vv_half_kick_device(x, v, f, m, dt, box, move=True)
                    if constraints is not None:
                        settle_device(x_old, x, v, constraints, m_o, m_h, dt, box)
                state.step += 1
            report = state.step % report_interval == 0 or state.step == n_steps
            with timer.section("lifecycle"):
                interval_due = state.step - state.plist.build_step >= policy.rebuild_interval
                guard_due = False
                speculative = False
                # d_max grows about linearly between rebuilds: when this step's
                # extrapolated value would fire the guard, a speculative pass
                # would likely be thrown away -- read d_max first instead
                likely = 2.0 * (2.0 * d_max - d_last) > buffer
                d_last = d_max
                if not interval_due and likely:
                    d_max = max(d_max, float(max_displacement_device(ref, x, box).item()))
                    guard_due = 2.0 * d_max > buffer
                elif not interval_due:
                    # drift guard without stalling the GPU: d_max goes to
                    # pinned memory ahead of a speculative force pass on the
                    # current list; the host reads it while that pass runs and,
                    # when the guard fires (rare), rebuilds and redoes the pass
                    # -- the reference's decision at the same step
                    d_pin.copy_(max_displacement_device(ref, x, box), non_blocking=True)
                    d_ev.record()
                    with timer.section("forces"):
                        force_pass(report)
                    speculative = True
                    d_ev.synchronize()
                    d_max = max(d_max, float(d_pin[0]))
                    guard_due = 2.0 * d_max > buffer
                if interval_due or guard_due:
                    speculative = False
                    if guard_due:
                        state.n_drift_rebuilds += 1
                    with timer.section("rebuild"):
                        # grid + search (+ exclusions) + prune + force layout in one
                        # native call: no interpreter time between the phases
                        state.grid, state.plist = list_step(
                            _DeviceSystem(system, x), state.grid.m, state.target_occupancy, box, params.r_list,
                            positions=x, r_inner=min(policy.r_inner, params.r_list),
                            prune=policy.prune_on_build and policy.rebuild_interval > 1, molecules=mol,
                            supercluster_size=state.plist.supercluster_size, n_lane=state.plist.n_lane,
                            build_step=state.step)
                    ref.copy_(x)
                    d_max = d_last = 0.0
                    state.n_rebuilds += 1
            if not speculative:
                with timer.section("forces"):
                    force_pass(report)
            with timer.section("integrate"):
                if fused:  # half kick + RATTLE in one kernel
                    vv_constrained_device(x, v, f, m, constraints, m_o, m_h, dt, box, phase=1)
                else:
                    vv_half_kick_device(x, v, f, m, dt, box, move=False)
                    if constraints is not None:
                        settle_device(None, x, v, constraints, m_o, m_h, dt, box, velocities_only=True)
            if report:
                with timer.section("report"):
                    record()
    torch.cuda.synchronize()
    state.system = replace(system, positions=x.cpu().numpy(), velocities=v.cpu().numpy())
    state.drift = DriftTracker(reference_positions=ref.cpu().numpy(), max_displacement=d_max)
    eh = e.cpu().numpy()
    forces = ForcesEnergies(forces=f.cpu().numpy(), e_lj=float(eh[0]), e_coulomb=float(eh[1]))
    wall = time.perf_counter() - wall0
    res = RunResult(state=state, forces=forces, steps=np.asarray(steps, dtype=np.int64), e_kinetic=np.asarray(e_kin),
                    e_potential=np.asarray(e_pot), temperature=np.asarray(temps), max_drift=np.asarray(drifts),
                    timing=timer, wall_seconds=wall, log_lines=log)
    dev_abs, dev_rel = res.energy_drift()
    log.append(f"# energy drift: abs={dev_abs:.6e} kJ/mol rel={dev_rel:.6e}")
    return res


class _DeviceSystem:
    """The ParticleSystem fields build_cluster_grid reads (n, box), with the
    positions supplied separately as a device tensor."""

    def __init__(self, system: ParticleSystem, positions: torch.Tensor):
        self.n = system.n
        self.box = system.box
        self.positions = positions
