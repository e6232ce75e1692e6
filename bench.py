"""Benchmark: nbnxn search + force on synthetic SPC water (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--atoms 96000] [--elec ewald|rf|cutoff] [--nstlist 10] [--rlist 1.1]
                    [--positions moving|static] [--rinner R]

One STEP = one MD step of the non-bonded hot path on MOVING positions
(default): the atoms follow a deterministic trajectory (every water molecule
oscillates rigidly about its start with amplitude 0.025 nm and a period of
40-80 steps: an MD stand-in -- the reference's SPC water has no exclusions or
constraints, so real dynamics of it diverge), the list
lifecycle of run_md runs on the device (rebuild -- grid, cluster-pair search,
prune from scratch -- every nstlist steps or when the drift guard
2 d_max > r_list - r_c fires, one scalar read per step), and every step runs
the force pass (energies every nstlist steps).  --positions static keeps the
box fixed (the r01 configuration).

value   = useful pair interactions (admitted slot pairs with r <= r_c) per
          second, whole job, inputs resident in HBM, per-step CUDA events,
          L2 flushed (256 MiB write) between steps outside the timed events.
e2e     = the same metric through the drop-in API a reference user calls:
          compute_nonbonded_original with numpy host arrays every step,
          build_cluster_grid / build_pair_list / prune_pair_list on a
          ParticleSystem every nstlist steps; wall clock per step (host
          conversions, H2D of positions / charges / types, D2H of forces and
          energies included).  e2e_pinned: the device API with pinned host
          buffers copied in and out every step (CUDA events).
roofline= the force kernel (k_force) against the FP32 pipe peak
          (148 SMs x 128 lanes x 2 flop x sm_max_mhz from MEASURED_PEAKS.json),
          flops = admitted slot pairs the kernel evaluates x per-pair cost
          (kernels.FLOPS_PER_PAIR = 40, +12 for Ewald), kernel time from
          CUDA events around every launch of K force passes on the moved
          positions.  Dynamic pruning (--rinner > 0) is off by default for
          moving positions (the inner list is invalidated within a few steps
          of motion) and r_c + 0.02 nm for static ones.
cpu_baseline = the reference algorithm's CPU port (oracle/, FP64, all host
          threads) on the same system: one rebuild + one force pass.
--impl reference: that CPU port timed for W + K steps of the same
          trajectory (rank 0 only).
"""

from __future__ import annotations

import argparse
import faulthandler
import gc
import json
import os
import statistics
import sys
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parent
sys.path.insert(0, str(REPO))

DT_PS = 0.002
R_CUT, R_LIST, M = 1.0, 1.1, 4


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--atoms", type=int, default=96000)
    ap.add_argument("--elec", default="ewald", choices=["ewald", "rf", "cutoff"])
    ap.add_argument("--nstlist", type=int, default=10)
    ap.add_argument("--rlist", type=float, default=1.1, help="buffered list cutoff r_list in nm (config 5 sweep)")
    ap.add_argument("--rinner", type=float, default=None,
                    help="dynamic-pruning inner radius in nm (default: off for moving positions, r_c + 0.02 "
                         "for static; 0 = off)")
    ap.add_argument("--positions", default="moving", choices=["moving", "static"])
    ap.add_argument("--occupancy", default="tuned", choices=["tuned", "default"])
    ap.add_argument("--m", type=int, default=4, choices=[4, 8], help="cluster size (4x4 or 8x8 cluster pairs)")
    ap.add_argument("--migrate", action="store_true",
                    help="N > 1: list steps by neighbour-only particle migration (SlabDecomposition.migrate) "
                         "instead of the all-gather of home positions")
    ap.add_argument("--slabs", default="count", choices=["count", "equal"],
                    help="N > 1: initial slab boundaries (equal particle counts, or equal widths)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-md", action="store_true", help="skip the rigid-water run_md ns/day measurement")
    ap.add_argument("--md-steps", type=int, default=200)
    ap.add_argument("--balance", action="store_true",
                    help="N > 1: rebalance the slabs from the ranks' force times at every rebuild (off: on the "
                         "uniform water box it only adds a sync + all-gather per rebuild, 0.999 vs 0.907 ms/step "
                         "at 1.5M on 4 B200)")
    return ap.parse_args()


def workload(args):
    from paper_1506_00716_b200.systems import spc_water, tuned_occupancy

    system, table = spc_water(args.atoms, seed=2024)
    L = float(system.box.lengths[0])
    occ = tuned_occupancy(args.atoms, L, M) if args.occupancy == "tuned" else None
    return system, table, occ


AMP_NM = 0.025  # trajectory amplitude: 10-step displacement <= 0.035 nm < (r_list - r_c) / 2


class Trajectory:
    """Deterministic MD stand-in: molecule m (atoms 3m..3m+2, rigid) moves as
    x0 + A (sin(w_m k + p_m) - sin(p_m)) u_m, u_m a random unit vector,
    w_m in [2 pi / 80, 2 pi / 40] per step.  x(0) = x0; any 10-step window
    moves an atom by at most 2 A sin(10 w / 2) < 0.035 nm, so interval
    rebuilds alone keep the list valid (the drift guard still runs)."""

    def __init__(self, system, static=False, seed=7):
        n = system.n
        rng = np.random.default_rng(seed)
        nmol = (n + 2) // 3
        u = rng.normal(size=(nmol, 3))
        u /= np.linalg.norm(u, axis=1, keepdims=True)
        self.u = np.repeat(u, 3, axis=0)[:n]
        self.w = np.repeat(rng.uniform(2 * np.pi / 80, 2 * np.pi / 40, nmol), 3)[:n]
        self.p = np.repeat(rng.uniform(0, 2 * np.pi, nmol), 3)[:n]
        self.x0 = np.array(system.positions)
        self.static = static

    def host(self, k):
        if self.static:
            return self.x0
        s = AMP_NM * (np.sin(self.w * k + self.p) - np.sin(self.p))
        return self.x0 + s[:, None] * self.u

    def to_device(self, dev, steps):
        """Materialise the positions of trajectory steps `steps` in HBM (the
        stand-in for the integrator's output: no per-step kernel)."""
        import torch

        self.dev_pos = {k: torch.from_numpy(self.host(k)).to(dev) for k in steps}

    def device(self, k, out=None):
        """positions of step k (device tensor)."""
        return self.dev_pos[k]


def make_params(args, table):
    import paper_1506_00716_b200 as nbx

    if args.elec == "ewald":
        return nbx.NonbondedParams(r_cut=R_CUT, r_list=R_LIST, lj_table=table, shift_potential=True,
                                   elec="ewald", ewald_beta=nbx.ewald_beta(R_CUT, 1e-5))
    if args.elec == "rf":
        return nbx.NonbondedParams(r_cut=R_CUT, r_list=R_LIST, lj_table=table, shift_potential=True,
                                   elec="reaction_field", epsilon_rf=0.0)
    return nbx.NonbondedParams(r_cut=R_CUT, r_list=R_LIST, lj_table=table, shift_potential=True)


def workload_name(args):
    elec = {"ewald": "Ewald real-space (erfc, beta: erfc(beta rc)=1e-5)", "rf": "reaction-field (eps_rf=inf)",
            "cutoff": "shifted cutoff Coulomb (= RF eps_rf=1, reference physics)"}[args.elec]
    return f"SPC water {args.atoms // 1000}k atoms, LJ+{elec}"


def positions_note(args):
    if args.positions == "static":
        return "static (search+prune from scratch every nstlist steps, forces every step, energies every nstlist steps)"
    return (f"moving: rigid molecules oscillating about their start (amplitude {AMP_NM} nm, period 40-80 steps; "
            "MD stand-in); list rebuilt from scratch every nstlist steps or when the drift guard fires, "
            "forces every step, energies every nstlist steps")


def config(args, occ, extra=None):
    """config of our arm (GPU)."""
    c = {"workload": workload_name(args),
         "n_atoms": args.atoms, "r_cut_nm": R_CUT, "r_list_nm": R_LIST, "cluster_size": M,
         "nstlist": args.nstlist, "r_inner_nm": getattr(args, "rinner", 0.0) or 0.0,
         "grid_occupancy": args.occupancy if occ is None else f"tuned ({occ:.1f})",
         "positions": positions_note(args),
         "dynamic_pruning": ("off" if not getattr(args, "rinner", 0.0) else
                             "inner force list at r_inner, used while 2 d_max <= r_inner - r_c (device check per call)"),
         "l2": "flushed between steps by a 256 MiB write outside the timed events",
         "parallelism": f"{'slab DD' if args.gpus > 1 else 'single GPU'} x{args.gpus}"}
    if extra:
        c.update(extra)
    return c


def config_reference(args, occ, threads):
    """config of the reference arm: the oracle's C port of the reference CPU
    path -- no dynamic pruning, no GPU, no cache flush."""
    return {"workload": workload_name(args), "n_atoms": args.atoms, "r_cut_nm": R_CUT, "r_list_nm": R_LIST,
            "cluster_size": M, "nstlist": args.nstlist,
            "grid_occupancy": args.occupancy if occ is None else f"tuned ({occ:.1f})",
            "positions": positions_note(args),
            "impl": ("oracle/ C port of the reference CPU path (FP64; grid numpy, O(n_c^2) search, prune and "
                     f"blocked force kernel in C with OpenMP on {threads} host threads)"),
            "parallelism": f"CPU x{threads} threads"}


# ---------------------------------------------------------------- clocks
class Clocks:
    """SM clock + clock-event reasons sampled through NVML every ~5 ms on a
    background thread while the timed region runs (also one sample at start
    and one at stop, so short multi-rank regions always have records).  The
    NVML device is the one this rank's CUDA device maps to (by UUID)."""

    REASONS = {"hw_slowdown": "nvmlClocksEventReasonHwSlowdown",
               "hw_thermal_slowdown": "nvmlClocksEventReasonHwThermalSlowdown",
               "sw_thermal_slowdown": "nvmlClocksEventReasonSwThermalSlowdown",
               "sw_power_cap": "nvmlClocksEventReasonSwPowerCap"}

    def __init__(self, idx):
        import threading

        self.samples, self.reasons, self.max_mhz = [], set(), 0.0
        self.h = None
        try:
            import pynvml
            import torch

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = self._handle(pynvml, torch, idx)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM))
        except Exception:
            self.h = None
            return
        self._stop = threading.Event()
        self._sample()
        self.th = None
        if os.environ.get("NBX_BENCH_CLOCK_THREAD", "1") != "0":  # 0: samples at start and stop only (A/B)
            self.th = threading.Thread(target=self._run, daemon=True)
            self.th.start()

    @staticmethod
    def _handle(nv, torch, idx):
        """NVML handle of CUDA device idx: matched by UUID (robust to
        CUDA_VISIBLE_DEVICES and to the enumeration order)."""
        want = str(torch.cuda.get_device_properties(idx).uuid).lower()
        want = want[4:] if want.startswith("gpu-") else want
        for i in range(nv.nvmlDeviceGetCount()):
            h = nv.nvmlDeviceGetHandleByIndex(i)
            u = nv.nvmlDeviceGetUUID(h)
            u = (u.decode() if isinstance(u, bytes) else str(u)).lower()
            if (u[4:] if u.startswith("gpu-") else u) == want:
                return h
        return nv.nvmlDeviceGetHandleByIndex(idx)

    def _sample(self):
        nv = self.nv
        self.samples.append(float(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)))
        bits = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        for name, const in self.REASONS.items():
            if bits & getattr(nv, const):
                self.reasons.add(name)

    def _run(self):
        while not self._stop.wait(0.005):
            try:
                self._sample()
            except Exception:
                return

    def stop(self):
        if self.h is None:
            return None
        self._stop.set()
        if self.th is not None:
            self.th.join()
        self._sample()
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples), "source": "nvml"}


# ---------------------------------------------------------------- CPU port
def cpu_port_times(system, params_phys, occ, nstlist, reps=1):
    """Reference algorithm (oracle/, FP64): numpy grid, O(n_c^2) AABB search
    (pairlist.py:185-189), prune, and the blocked force kernel (kernels.py:124-221)
    on all host threads."""
    from oracle import native, search

    L = system.box.lengths
    threads = native.default_threads()
    t0 = time.perf_counter()
    og = search.build_grid(system.positions, L, M, occ)
    t1 = time.perf_counter()
    ol = native.search_list(og, L, R_LIST, method="n2", threads=threads)
    t2 = time.perf_counter()
    op = native.prune_list(ol, og["clustered_positions"], L, threads=threads)
    t3 = time.perf_counter()
    bits = np.ascontiguousarray(search.pack_masks(op["masks"]))
    tf = []
    for _ in range(reps):
        t4 = time.perf_counter()
        native.list_forces(op, og, system.positions, system.charges, system.lj_type, L, params_phys,
                           threads=threads, packed_masks=bits)
        tf.append(time.perf_counter() - t4)
    return dict(grid=t1 - t0, search=t2 - t1, prune=t3 - t2, force=min(tf), threads=threads, og=og, op=op)


def oracle_physics(params):
    from oracle import forces as of

    return of.Physics(r_cut=params.r_cut, lj_table=params.lj_table, coulomb_scale=params.coulomb_scale,
                      shift_potential=params.shift_potential, elec=params.elec,
                      epsilon_rf=params.epsilon_rf, ewald_beta=params.ewald_beta)


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    system, table, occ = workload(args)
    params = make_params(args, table)
    phys = oracle_physics(params)
    from oracle import native, search

    L = system.box.lengths
    threads = native.default_threads()
    traj = Trajectory(system, static=args.positions == "static")
    state = {}
    within = []

    def step(k, count=False):
        pos = traj.host(k)
        if k % args.nstlist == 0 or not state:
            og = search.build_grid(pos, L, M, occ)
            ol = native.search_list(og, L, R_LIST, method="n2", threads=threads)
            op = native.prune_list(ol, og["clustered_positions"], L, threads=threads)
            state.update(og=og, op=op, bits=np.ascontiguousarray(search.pack_masks(op["masks"])))
            if count:
                within.append(native.count_within(op, og["clustered_positions"], L, R_CUT, threads=threads))
        native.list_forces(state["op"], state["og"], pos, system.charges, system.lj_type, L, phys,
                           threads=threads, packed_masks=state["bits"])

    for k in range(args.warmup):
        step(k)
    t0 = time.perf_counter()
    for k in range(args.warmup, args.warmup + args.steps):
        step(k, count=True)
    dt = time.perf_counter() - t0
    if not within:  # no rebuild inside the timed steps
        within.append(native.count_within(state["op"], state["og"]["clustered_positions"], L, R_CUT, threads=threads))
    n_within = float(np.mean(within))
    value = n_within * args.steps / dt
    line = {
        "impl": "reference", "metric": "nonbonded pair-interactions/s (useful, r<=r_c)", "value": value,
        "unit": "pairs/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * dt / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "ns_per_day": args.steps / dt * DT_PS * 86.4,
        "config": config_reference(args, occ, threads),
        "cpu_baseline": {"value": value, "unit": "pairs/s", "cores": threads, "kind": "port",
                         "sample": f"{args.steps} steps (rebuild every {args.nstlist}) of the full workload"},
        "e2e": {"value": value, "unit": "pairs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- rigid-water MD
def rigid_water_md(args, params, occ):
    """ns/day of real dynamics on the benchmark box: engine.run_md with
    RigidWater (SETTLE + RATTLE, intramolecular exclusions), NVE velocity
    Verlet at 2 fs, energies every nstlist steps, the run_md list lifecycle
    (interval + drift guard).  The generated lattice is first relaxed and
    brought to 300 K (five 20-step runs with velocity rescaling between them,
    untimed); the timed run's wall clock excludes its one-time setup."""
    import dataclasses

    import torch

    import paper_1506_00716_b200 as nbx
    from paper_1506_00716_b200.systems import spc_water

    system, _ = spc_water(args.atoms, seed=2024, temperature=300.0)
    water = nbx.RigidWater()
    layout = nbx.KernelLayout(M, M)
    dt = DT_PS
    for _ in range(5):
        res = nbx.run_md(system, params, layout, dt, 20, report_interval=20, target_occupancy=occ,
                         constraints=water)
        v = res.state.system.velocities * np.sqrt(300.0 / max(float(res.temperature[-1]), 1.0))
        system = dataclasses.replace(res.state.system, velocities=v)
    n_steps = args.md_steps
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = nbx.run_md(system, params, layout, dt, n_steps, report_interval=args.nstlist, target_occupancy=occ,
                     constraints=water)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0 - res.timing.total("setup")
    e = res.e_total
    ke = float(np.mean(res.e_kinetic))
    return {"ns_per_day": n_steps / wall * dt * 86.4, "steps": n_steps, "dt_ps": dt, "ms_per_step": 1e3 * wall / n_steps,
            "temperature_K": [round(float(res.temperature[0]), 1), round(float(res.temperature[-1]), 1)],
            "rebuilds": res.state.n_rebuilds, "drift_rebuilds": res.state.n_drift_rebuilds,
            "energy_excursion_over_ke": float(np.abs(e - e[0]).max() / ke),
            "timing": "host wall clock of run_md after its setup (per-step host sync: one d_max read)",
            "system": f"{args.atoms // 3} rigid SPC waters, {workload_name(args).split(', ', 1)[1]}"}


# ---------------------------------------------------------------- GPU arm
def run_ours(args):
    import torch

    import paper_1506_00716_b200 as nbx
    from paper_1506_00716_b200 import _lib
    from paper_1506_00716_b200.engine import max_displacement_device
    from paper_1506_00716_b200.kernels import flops_per_pair

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        return run_dd(args, world, rank, local)
    lib = _lib.load()
    system, table, occ = workload(args)
    params = nbx.NonbondedParams(**{k: getattr(make_params(args, table), k) for k in (
        "r_cut", "r_list", "lj_table", "coulomb_scale", "shift_potential", "elec", "epsilon_rf", "ewald_beta")})
    box = system.box
    n = system.n
    dev = torch.device("cuda", local)
    W = max(3, args.warmup)
    S0 = 10 * args.nstlist  # first timed step (trajectory index)
    n_setup = 2 * args.nstlist if args.nstlist <= 50 else 2
    traj = Trajectory(system, static=args.positions == "static")
    traj.to_device(dev, sorted(set(range(n_setup)) | set(range(S0 - W, S0 + args.steps))))
    ref_d = torch.empty((n, 3), dtype=torch.float64, device=dev)  # build positions (drift-guard reference)
    q_d = torch.from_numpy(np.array(system.charges)).to(dev)
    t_d = torch.from_numpy(np.array(system.lj_type)).to(dev)
    f_d = torch.empty((n, 3), dtype=torch.float64, device=dev)
    e_d = torch.zeros(2, dtype=torch.float64, device=dev)
    bad_d = torch.empty(2, dtype=torch.int64, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    buffer = R_LIST - R_CUT
    st = {}

    def rebuild(k, pos, counts):
        grid, plist = nbx.list_step(system, M, occ, box, R_LIST, positions=pos, r_inner=args.rinner)
        st.update(grid=grid, plist=plist, build=k, rebuilds=st.get("rebuilds", 0) + 1)
        ref_d.copy_(pos)
        if counts is not None:
            counts[k] = nbx.interaction_stats(plist, grid, grid.clustered_positions_device, box, R_CUT).n_within_cutoff

    d_pin = torch.zeros(1, dtype=torch.float64).pin_memory()
    d_ev = torch.cuda.Event()

    def force(k, pos, q, t, out):
        nbx.compute_nonbonded_device(st["plist"], st["grid"], pos, q, t, params, box,
                                     energy=(k % args.nstlist == 0), out=out, e_out=e_d, bad=bad_d)

    def step(k, q, t, out, counts=None):
        """one MD step of the hot path: positions of step k, list lifecycle
        (interval or drift guard 2 d_max > r_list - r_c, engine.lifecycle_tick),
        force pass.  The drift guard is evaluated without stalling the GPU:
        d_max is reduced and copied to pinned memory ahead of a speculative
        force pass on the current list, and the host reads it while that pass
        runs; when the guard fires (rare) the list is rebuilt and the pass
        redone -- the same decision, at the same step, as the reference."""
        pos = traj.device(k)
        due = "plist" not in st or k - st["build"] >= args.nstlist
        if due:
            rebuild(k, pos, counts)
            force(k, pos, q, t, out)
            return
        if traj.static:
            force(k, pos, q, t, out)
            return
        d_pin.copy_(max_displacement_device(ref_d, pos, box), non_blocking=True)
        d_ev.record()
        force(k, pos, q, t, out)
        d_ev.synchronize()
        if 2.0 * float(d_pin[0]) > buffer:
            st["drift"] = st.get("drift", 0) + 1
            rebuild(k, pos, counts)
            force(k, pos, q, t, out)

    # setup (not timed, not counted as warm-up steps): two list cycles so the
    # stream-ordered memory pool holds two list generations (steady state)
    for k in range(n_setup):
        step(k, q_d, t_d, f_d)
    # counting pass over exactly the timed steps (same rebuild schedule: the
    # lifecycle restarts at S0 - W in both passes): within-r_c pairs of every
    # list the timed pass will use
    counts = {}
    st.clear()
    for k in range(S0 - W, S0 + args.steps):
        step(k, q_d, t_d, f_d, counts=counts)
    torch.cuda.synchronize()
    if int(bad_d[0].item()) != -1:
        raise RuntimeError("singular pair in the benchmark system")
    builds = sorted(counts)
    within_at = [counts[max(b for b in builds if b <= k)] for k in range(S0, S0 + args.steps)]
    n_within_total = float(sum(within_at))
    n_admitted = nbx.interaction_stats(st["plist"], st["grid"], st["grid"].clustered_positions_device, box,
                                       R_CUT).n_admitted
    drift_count = st.get("drift", 0)

    # ---- device-resident timed region
    clocks = Clocks(local)
    st.clear()
    for k in range(S0 - W, S0):
        step(k, q_d, t_d, f_d)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    launches0 = lib.nbx_launch_count()
    gc.collect()  # no interpreter GC pause inside the timed region (re-enabled below)
    gc.disable()
    torch.cuda.synchronize()
    wall0 = time.perf_counter()
    for i in range(args.steps):
        flush.zero_()
        ev[i][0].record()
        step(S0 + i, q_d, t_d, f_d)
        ev[i][1].record()
    torch.cuda.synchronize()
    wall = time.perf_counter() - wall0
    gc.enable()
    launches = lib.nbx_launch_count() - launches0
    rebuilds_timed = st.get("rebuilds", 0)
    t_ms = float(sum(a.elapsed_time(b) for a, b in ev))
    if os.environ.get("NBX_BENCH_DEBUG"):
        print("per-step ms:", [round(a.elapsed_time(b), 3) for a, b in ev], file=sys.stderr)
    value = n_within_total / (t_ms * 1e-3)

    # ---- k_force duration: events around every launch of K force passes
    # (no energies) on the launching stream, same list, last timed positions
    lib.nbx_timing_enable(0)
    lib.nbx_timing_query(None, None)
    lib.nbx_timing_enable(1)
    pos_d = traj.device(S0 + args.steps - 1)
    for _ in range(args.steps):
        flush.zero_()
        nbx.compute_nonbonded_device(st["plist"], st["grid"], pos_d, q_d, t_d, params, box, energy=False,
                                     out=f_d, e_out=e_d, bad=bad_d)
    torch.cuda.synchronize()
    lib.nbx_timing_enable(0)
    fk_ms, fk_n = (np.zeros(1), np.zeros(1, dtype=np.int64))
    _lib.check(lib.nbx_timing_query(_lib.ptr(fk_ms), _lib.ptr(fk_n)), "timing")
    clk = clocks.stop()
    # pairs that launch evaluated: the inner list only while it is valid at
    # these positions (the kernel's own device test, 2 d_max <= r_inner - r_c)
    d_now = float(max_displacement_device(ref_d, pos_d, box).item())
    inner_ok = bool(args.rinner) and 2.0 * d_now <= args.rinner - R_CUT - 1e-4
    n_force = st["plist"].force_pairs(inner=inner_ok)

    # ---- e2e through the drop-in API (numpy host arrays, wall clock per step)
    layout = nbx.KernelLayout(M, M)
    # warm-up: W steps plus two whole list cycles before them (same rebuild
    # phase as the counting pass): the first two list steps of a fresh
    # drop-in loop run ~1.7 ms slower (one-time host / pool set-up)
    E0 = S0 - W - 2 * args.nstlist
    host_pos = [traj.host(k) for k in range(E0, S0 + args.steps)]
    charges, types = np.array(system.charges), np.array(system.lj_type)
    de = {}
    e2e_s = []
    h2d = d2h = 0
    gc.collect()  # interpreter GC paused during the loop, as in the device-timed regions
    gc.disable()
    for i, k in enumerate(range(E0, S0 + args.steps)):
        pos_np = host_pos[i]
        t0 = time.perf_counter()
        rb = "plist" not in de or k - de["build"] >= args.nstlist
        if rb:
            sysk = nbx.ParticleSystem(positions=pos_np, velocities=system.velocities, masses=system.masses,
                                      charges=charges, lj_type=types, box=box)
            grid = nbx.build_cluster_grid(sysk, M, occ)
            plist = nbx.prune_pair_list(nbx.build_pair_list(grid, box, R_LIST), grid.clustered_positions, box)
            de.update(grid=grid, plist=plist, build=k)
        res = nbx.compute_nonbonded_original(de["plist"], de["grid"], pos_np, charges, types, params, box, layout)
        dt = time.perf_counter() - t0
        if k >= S0:
            e2e_s.append(dt)
            h2d += 40 * n + (24 * n if rb else 0)
            d2h += 24 * n + 32 + (24 * de["grid"].n_slots if rb else 0)
    gc.enable()
    del res
    e2e_time = sum(e2e_s)
    if os.environ.get("NBX_BENCH_DEBUG"):
        print("e2e per-step ms:", [round(1e3 * x, 3) for x in e2e_s], file=sys.stderr)

    # ---- e2e with the device API and pinned host buffers (CUDA events)
    pin_pos = [torch.from_numpy(p).pin_memory() for p in host_pos]
    q_h = torch.from_numpy(np.array(charges)).pin_memory()  # (the drop-in call froze them in place)
    t_h = torch.from_numpy(np.array(types)).pin_memory()
    f_h = torch.empty((n, 3), dtype=torch.float64).pin_memory()
    e_h = torch.empty(2, dtype=torch.float64).pin_memory()
    q_s, t_s = torch.empty_like(q_d), torch.empty_like(t_d)
    st.clear()
    ev2 = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]

    pos_s = torch.empty((n, 3), dtype=torch.float64, device=dev)

    class Pinned:  # trajectory replay from pinned host memory (H2D inside the step)
        static = traj.static

        @staticmethod
        def device(k, out=None):
            return pos_s.copy_(pin_pos[k - E0], non_blocking=True)

    traj_dev = traj
    traj = Pinned
    for i, k in enumerate(range(S0 - W, S0 + args.steps)):
        if k >= S0:
            flush.zero_()
            ev2[i - W][0].record()
        q_s.copy_(q_h, non_blocking=True)
        t_s.copy_(t_h, non_blocking=True)
        step(k, q_s, t_s, f_d)
        f_h.copy_(f_d, non_blocking=True)
        e_h.copy_(e_d, non_blocking=True)
        if k >= S0:
            ev2[i - W][1].record()
    torch.cuda.synchronize()
    traj = traj_dev
    pin_ms = float(sum(a.elapsed_time(b) for a, b in ev2))

    # ---- roofline (force kernel, FP32 pipe)
    peaks = json.loads((REPO / "MEASURED_PEAKS.json").read_text()) if (REPO / "MEASURED_PEAKS.json").exists() else {}
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
    peak_tf = n_sm * 128 * 2 * sm_max * 1e6 / 1e12
    fpp = flops_per_pair(params)
    fk_avg_ms = float(fk_ms[0]) / max(1, int(fk_n[0]))
    achieved = n_force * fpp / (fk_avg_ms * 1e-3) / 1e12
    traffic = None
    prof = REPO / "profiles" / "force_kernel_ncu.json"
    if prof.exists():
        try:
            traffic = json.loads(prof.read_text()).get("dram_bytes_per_launch")
        except Exception:
            traffic = None

    line = {
        "metric": "nonbonded pair-interactions/s (useful, r<=r_c)",
        "value": value, "unit": "pairs/s", "n_gpus": world, "steps": args.steps, "warmup": W,
        "ms_per_step": t_ms / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "fp32 (pair math; fp64 energy + final force accumulation)",
        "data": "synthetic (seeded SPC-geometry water, BASELINE.md recipe; moving-trajectory stand-in)",
        "config": config(args, occ),
        "ns_per_day": args.steps / (t_ms * 1e-3) * DT_PS * 86.4,
        "ns_per_day_note": "steps/s of the timed hot-path loop x 2 fs (force + list lifecycle on the moving "
                           "stand-in trajectory; no integrator, SURVEY 0.3)",
        "pairs_per_step": {"within_rc": n_within_total / args.steps, "admitted": n_admitted,
                           "force_kernel": n_force, "admitted_per_s": n_admitted * args.steps / (t_ms * 1e-3)},
        "lifecycle": {"rebuilds_timed": rebuilds_timed, "drift_rebuilds_count_pass": drift_count},
        "e2e": {"value": n_within_total / e2e_time, "unit": "pairs/s", "kind": (
                    "drop-in API, numpy host arrays: compute_nonbonded_original every step, "
                    "build_cluster_grid/build_pair_list/prune_pair_list every nstlist; wall clock, interpreter GC paused"),
                "h2d_bytes_per_step": h2d // args.steps, "d2h_bytes_per_step": d2h // args.steps,
                "ms_per_step": 1e3 * e2e_time / args.steps},
        "e2e_pinned": {"value": n_within_total / (pin_ms * 1e-3), "unit": "pairs/s",
                       "kind": "device API, pinned host buffers copied in/out every step; CUDA events",
                       "h2d_bytes_per_step": 40 * n, "d2h_bytes_per_step": 24 * n + 16,
                       "ms_per_step": pin_ms / args.steps},
        "gpu_launches": int(launches),
        "roofline": {"bound": "fp32", "kernel": "k_force", "achieved": achieved, "peak": peak_tf,
                     "unit": "TFLOP/s", "frac": achieved / peak_tf, "traffic": traffic,
                     "kernel_ms": fk_avg_ms, "flops_per_pair": fpp,
                     "pairs": "force_kernel (admitted pairs the kernel evaluates)",
                     "peak_note": f"nominal FP32: {n_sm} SMs x 128 lanes x 2 x {sm_max:.0f} MHz (sm_max_mhz of MEASURED_PEAKS.json)"},
        "clocks": clk,
        "wall_s_timed": wall,
    }
    if not args.no_md:
        md = rigid_water_md(args, params, occ)
        line["md"] = md
        line["ns_per_day_hot_path"] = line["ns_per_day"]
        line["ns_per_day"] = md["ns_per_day"]
        line["ns_per_day_note"] = ("run_md: NVE velocity Verlet of the SPC box as rigid water (SETTLE + RATTLE, "
                                   "intramolecular exclusions), 2 fs, the same non-bonded path; see md")
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        c = cpu_port_times(system, oracle_physics(params), occ, args.nstlist)
        per_step = c["force"] + (c["grid"] + c["search"] + c["prune"]) / args.nstlist
        line["cpu_baseline"] = {
            "value": (n_within_total / args.steps) / per_step, "unit": "pairs/s", "cores": c["threads"], "kind": "port",
            "sample": (f"one rebuild (grid {c['grid']:.3f}s, O(n_c^2) search {c['search']:.3f}s, "
                       f"prune {c['prune']:.3f}s) + one force pass {c['force']:.3f}s, amortised over "
                       f"nstlist={args.nstlist}")}
    print(json.dumps(line), flush=True)


def run_dd(args, world, rank, local):
    """N > 1: strong scaling of the same box over N GPUs with the slab
    decomposition (paper_1506_00716_b200/dd.py): per step halo exchange
    (coordinates in, forces back: NVLink peer stores, NCCL fallback), local
    search every nstlist steps after an all-gather of the home positions
    (--migrate: neighbour-only particle migration instead),
    energies all-reduced on energy steps.  Positions follow the same moving
    trajectory as N = 1 (each rank takes its home rows of step k); lists are
    rebuilt every nstlist steps (the trajectory's 10-step displacement stays
    inside the buffer, so no cross-rank drift guard is needed)."""
    import datetime

    import torch
    import torch.distributed as dist

    import paper_1506_00716_b200 as nbx
    from paper_1506_00716_b200 import _lib
    from paper_1506_00716_b200.dd import DomainForces, SlabDecomposition
    from paper_1506_00716_b200.kernels import flops_per_pair

    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev, timeout=datetime.timedelta(seconds=120))
    lib = _lib.load()
    system, table, occ = workload(args)
    params = make_params(args, table)
    box = system.box
    W = max(3, args.warmup)
    S0 = 10 * args.nstlist
    n_setup = 2 * args.nstlist if args.nstlist <= 50 else 2
    traj = Trajectory(system, static=args.positions == "static")
    W2 = max(W, args.nstlist)  # the last warm-up covers a list step
    traj.to_device(dev, sorted(set(range(n_setup)) | set(range(S0 - W2, S0 + args.steps))))
    dd = SlabDecomposition(box.lengths, world, rank, r_comm=R_LIST)
    if args.slabs == "count":  # equal particle counts per slab at step 0 (same on every rank)
        dd.balance_counts(traj.host(0)[:, 0])
    dd.enable_native()
    p2p = dd.enable_p2p(system.n)  # per-step halo exchanges as NVLink peer stores (NBX_DD_P2P=0: NCCL)
    df = DomainForces(dd, system, params, M, occ, r_inner=args.rinner)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    lay = df.rebuild(traj.device(0))
    homes = {}
    balance = [args.balance]

    def step(k, home_pos=None, counts=None):
        nonlocal lay
        homes[k] = lay.home  # the home set whose step-k positions this rank supplies
        if home_pos is None:
            home_pos = traj.device(k).index_select(0, lay.home)
        if k % args.nstlist == 0:
            if args.migrate and not balance[0]:  # particles migrate to the neighbour slabs, no all-gather
                lay = df.rebuild_local(lay.home, home_pos)
            else:  # all-gather the home positions, re-assign (slabs rebalanced first with --balance)
                lay = df.rebuild(dd.allgather_home(lay.home, home_pos, system.n), balance=balance[0])
            if counts is not None:
                counts[k] = nbx.interaction_stats(df.plist, df.grid, df.grid.clustered_positions_device, box,
                                                  R_CUT).n_within_cutoff
        else:
            df.local_pos[:lay.n_home].copy_(home_pos)
        return df.forces(energy=(k % args.nstlist == 0))

    for k in range(n_setup):  # setup: memory pool steady state
        step(k)
    counts = {}
    for k in range(S0 - W, S0 + args.steps):  # counting pass over the timed steps (same rebuilds)
        step(k, counts=counts)
    torch.cuda.synchronize()
    builds = sorted(counts)
    within = [counts[max(b for b in builds if b <= k)] for k in range(S0, S0 + args.steps)] if builds else [0]
    cnt = torch.tensor([float(sum(within))], dtype=torch.float64, device=dev)
    dist.all_reduce(cnt)
    n_within_total = float(cnt.item())
    st = nbx.interaction_stats(df.plist, df.grid, df.grid.clustered_positions_device, box, R_CUT)
    adm = torch.tensor([st.n_admitted], dtype=torch.int64, device=dev)
    dist.all_reduce(adm)
    n_admitted = int(adm.item())
    n_force_rank = df.plist.force_pairs(inner=bool(args.rinner))  # this rank's kernel work
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    clocks = Clocks(local)
    gc.collect()  # no interpreter GC pause inside the timed region (re-enabled below)
    gc.disable()
    # warm-up after the set-up above and over a whole list cycle: the first
    # step after it (a list step) now and then stalled all ranks for 20-30 ms
    for k in range(S0 - W2, S0):
        step(k)
    lib.nbx_timing_query(None, None)
    lib.nbx_timing_enable(1)
    launches0 = lib.nbx_launch_count()
    dist.barrier()
    torch.cuda.synchronize()
    for i in range(args.steps):
        flush.zero_()
        ev[i][0].record()
        step(S0 + i)
        ev[i][1].record()
    torch.cuda.synchronize()
    gc.enable()
    launches = lib.nbx_launch_count() - launches0
    lib.nbx_timing_enable(0)
    fk_ms, fk_n = np.zeros(1), np.zeros(1, dtype=np.int64)
    _lib.check(lib.nbx_timing_query(_lib.ptr(fk_ms), _lib.ptr(fk_n)), "timing")
    clk = clocks.stop()
    if os.environ.get("NBX_BENCH_DEBUG"):
        print(f"rank {rank} per-step ms:", [round(a.elapsed_time(b), 3) for a, b in ev], file=sys.stderr)
    t = torch.tensor([sum(a.elapsed_time(b) for a, b in ev)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_ms = float(t.item())
    clk_all = [None] * world
    dist.all_gather_object(clk_all, clk)
    # e2e: this rank's home positions of step k H2D from pinned host memory,
    # home forces + energies D2H, every step.  The slab boundaries are frozen
    # for this phase and an untimed dry pass records the home set each step
    # starts from, so the timed replay feeds exactly those rows.
    balance[0] = False
    for k in range(S0 - W, S0 + args.steps):
        step(k)
    torch.cuda.synchronize()
    host_home = {k: torch.from_numpy(traj.host(k)[homes[k].cpu().numpy()]).pin_memory()
                 for k in range(S0 - W, S0 + args.steps)}
    ev2 = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    bytes_io = torch.zeros(2, dtype=torch.int64, device=dev)
    gc.collect()
    gc.disable()
    for i, k in enumerate(range(S0 - W, S0 + args.steps)):
        if i >= W:
            flush.zero_()
            ev2[i - W][0].record()
        hp = host_home[k].to(dev, non_blocking=True)
        f, e = step(k, home_pos=hp)
        f_host = torch.empty(f.shape, dtype=f.dtype).pin_memory()
        f_host.copy_(f, non_blocking=True)
        e.to("cpu", non_blocking=True)
        if i >= W:
            ev2[i - W][1].record()
            bytes_io[0] += hp.numel() * 8
            bytes_io[1] += f.numel() * 8 + 16
    torch.cuda.synchronize()
    gc.enable()
    t2 = torch.tensor([sum(a.elapsed_time(b) for a, b in ev2)], dtype=torch.float64, device=dev)
    dist.all_reduce(t2, op=dist.ReduceOp.MAX)
    dist.all_reduce(bytes_io)
    e2e_ms = float(t2.item())
    dd.check_p2p()  # a timed-out peer wait invalidates the run: raise instead of printing a line
    peaks = json.loads((REPO / "MEASURED_PEAKS.json").read_text()) if (REPO / "MEASURED_PEAKS.json").exists() else {}
    sm_max = float(peaks.get("sm_max_mhz", 1965.0))
    n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
    peak_tf = n_sm * 128 * 2 * sm_max * 1e6 / 1e12
    fk_avg_ms = float(fk_ms[0]) / max(1, int(fk_n[0]))
    achieved = n_force_rank * flops_per_pair(params) / (fk_avg_ms * 1e-3) / 1e12
    if rank == 0:
        good = [c for c in clk_all if c]
        clocks_line = None
        if good:
            clocks_line = {"sm_mhz": min(c["sm_mhz"] for c in good), "sm_max_mhz": max(c["sm_max_mhz"] for c in good),
                           "reasons": sorted(set(r for c in good for r in c["reasons"])),
                           "samples": sum(c["samples"] for c in good), "source": "nvml, all ranks (min median)"}
        line = {
            "metric": "nonbonded pair-interactions/s (useful, r<=r_c)",
            "value": n_within_total / (t_ms * 1e-3), "unit": "pairs/s", "n_gpus": world,
            "steps": args.steps, "warmup": W, "ms_per_step": t_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None,
            "dtype": "fp32 (pair math; fp64 energy + final force accumulation)",
            "data": "synthetic (seeded SPC-geometry water, BASELINE.md recipe; moving-trajectory stand-in)",
            "config": config(args, occ, {"parallelism": f"slab DD x{world} (half-shell halo, r_comm=r_list, "
                                                         f"{'NVLink peer stores' if p2p else 'NCCL send/recv'}, "
                                                         f"{'slabs rebalanced by force time at every rebuild' if args.balance else ('count-balanced slabs' if args.slabs == 'count' else 'equal slabs')})",
                                         "slab_boundaries_nm": [round(float(x), 4) for x in dd.boundaries]}),
            "ns_per_day": args.steps / (t_ms * 1e-3) * DT_PS * 86.4,
            "ns_per_day_note": "steps/s of the timed hot-path loop x 2 fs (no integrator)",
            "pairs_per_step": {"within_rc": n_within_total / args.steps, "admitted": n_admitted},
            "e2e": {"value": n_within_total / (e2e_ms * 1e-3), "unit": "pairs/s",
                    "kind": "device API per rank, pinned home positions in / home forces out every step; CUDA events",
                    "h2d_bytes_per_step": int(bytes_io[0].item()) // args.steps,
                    "d2h_bytes_per_step": int(bytes_io[1].item()) // args.steps, "ms_per_step": e2e_ms / args.steps},
            "gpu_launches": int(launches),
            "roofline": {"bound": "fp32", "kernel": "k_force (rank 0)", "achieved": achieved, "peak": peak_tf,
                         "unit": "TFLOP/s", "frac": achieved / peak_tf, "traffic": None, "kernel_ms": fk_avg_ms,
                         "flops_per_pair": flops_per_pair(params),
                         "pairs": "force_kernel of rank 0 (admitted pairs the kernel evaluates)"},
            "clocks": clocks_line,
        }
        print(json.dumps(line), flush=True)
    dist.barrier()
    dd.close()
    dist.destroy_process_group()


def main():
    global R_LIST, M
    faulthandler.enable()
    args = parse()
    R_LIST = args.rlist
    M = args.m
    if args.rinner is None:
        args.rinner = 0.0 if args.positions == "moving" else min(R_CUT + 0.02, R_LIST)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
