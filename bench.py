"""Benchmark: nbnxn search + force on synthetic SPC water (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--atoms 96000] [--elec ewald|rf|cutoff] [--nstlist 10] [--rlist 1.1]

One STEP = one MD step of the non-bonded hot path: every `nstlist` steps the
grid, the cluster-pair search and the prune are redone from scratch at the
current positions, and every step runs the force + energy pass.  Positions
are static (the reference's SPC water has no exclusions/constraints, so its
MD diverges -- SURVEY.md 0.3); nothing is cached across rebuilds.

value   = useful pair interactions (admitted slot pairs with r <= r_c) per
          second, whole job, inputs resident in HBM, per-step CUDA events,
          L2 flushed (256 MiB write) between steps outside the timed events.
e2e     = the same metric with host (pinned) positions/charges/types copied
          H2D and forces + energies copied D2H inside every timed step.
roofline= the force kernel (k_force) against the FP32 pipe peak
          (148 SMs x 128 lanes x 2 flop x sm_max_mhz from MEASURED_PEAKS.json),
          flops = admitted slot pairs the kernel evaluates x per-pair cost
          (kernels.FLOPS_PER_PAIR = 40, +12 for Ewald).  With dynamic
          pruning (--rinner, default r_c + 0.02 nm; 0 = off) those are the
          inner list's pairs (pairs_per_step.force_kernel), not the r_list
          list's (pairs_per_step.admitted).
cpu_baseline = the reference algorithm's CPU port (oracle/, FP64, all host
          threads) on the same system: one rebuild + one force pass.
--impl reference: that CPU port timed for W + K steps (rank 0 only).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
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
                    help="dynamic-pruning inner radius in nm (default r_c + 0.02; 0 = off)")
    ap.add_argument("--occupancy", default="tuned", choices=["tuned", "default"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def workload(args):
    from paper_1506_00716_b200.systems import spc_water, tuned_occupancy

    system, table = spc_water(args.atoms, seed=2024)
    L = float(system.box.lengths[0])
    occ = tuned_occupancy(args.atoms, L, M) if args.occupancy == "tuned" else None
    return system, table, occ


def make_params(args, table):
    import paper_1506_00716_b200 as nbx

    if args.elec == "ewald":
        return nbx.NonbondedParams(r_cut=R_CUT, r_list=R_LIST, lj_table=table, shift_potential=True,
                                   elec="ewald", ewald_beta=nbx.ewald_beta(R_CUT, 1e-5))
    if args.elec == "rf":
        return nbx.NonbondedParams(r_cut=R_CUT, r_list=R_LIST, lj_table=table, shift_potential=True,
                                   elec="reaction_field", epsilon_rf=0.0)
    return nbx.NonbondedParams(r_cut=R_CUT, r_list=R_LIST, lj_table=table, shift_potential=True)


def config(args, occ, extra=None):
    c = {"workload": f"SPC water {args.atoms // 1000}k atoms, LJ+{ {'ewald': 'Ewald real-space (erfc, beta: erfc(beta rc)=1e-5)', 'rf': 'reaction-field (eps_rf=inf)', 'cutoff': 'shifted cutoff Coulomb (= RF eps_rf=1, reference physics)'}[args.elec]}",
         "n_atoms": args.atoms, "r_cut_nm": R_CUT, "r_list_nm": R_LIST, "cluster_size": M,
         "nstlist": args.nstlist, "r_inner_nm": getattr(args, "rinner", 0.0) or 0.0, "grid_occupancy": args.occupancy if occ is None else f"tuned ({occ:.1f})",
         "positions": "static (search+prune from scratch every nstlist steps, forces every step, energies every nstlist steps)",
         "dynamic_pruning": ("off" if not getattr(args, "rinner", 0.0) else
                             "inner force list at r_inner, used while 2 d_max <= r_inner - r_c (device check per call)"),
         "l2": "flushed between steps by a 256 MiB write outside the timed events",
         "parallelism": f"{'replicas' if args.gpus > 1 else 'single'} x{args.gpus}"}
    if extra:
        c.update(extra)
    return c


# ---------------------------------------------------------------- clocks
class Clocks:
    def __init__(self, idx):
        self.proc = None
        self.path = REPO / "gpurun_out" / f"clocks_{os.getpid()}.csv"
        try:
            self.path.parent.mkdir(exist_ok=True)
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(idx), "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"], stdout=self.fh, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        self.proc.wait()
        self.fh.close()
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.path.read_text().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for name, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


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
    state = {}

    def step(k):
        if k % args.nstlist == 0 or not state:
            og = search.build_grid(system.positions, L, M, occ)
            ol = native.search_list(og, L, R_LIST, method="n2", threads=threads)
            op = native.prune_list(ol, og["clustered_positions"], L, threads=threads)
            state.update(og=og, op=op, bits=np.ascontiguousarray(search.pack_masks(op["masks"])))
        native.list_forces(state["op"], state["og"], system.positions, system.charges, system.lj_type, L, phys,
                           threads=threads, packed_masks=state["bits"])

    for k in range(args.warmup):
        step(k)
    n_within = native.count_within(state["op"], state["og"]["clustered_positions"], L, R_CUT, threads=threads)
    t0 = time.perf_counter()
    for k in range(args.warmup, args.warmup + args.steps):
        step(k)
    dt = time.perf_counter() - t0
    value = n_within * args.steps / dt
    line = {
        "impl": "reference", "metric": "nonbonded pair-interactions/s (useful, r<=r_c)", "value": value,
        "unit": "pairs/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * dt / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "ns_per_day": args.steps / dt * DT_PS * 86.4,
        "config": config(args, occ, {"impl": "oracle/ C port of the reference CPU path (no GPU)"}),
        "cpu_baseline": {"value": value, "unit": "pairs/s", "cores": threads, "kind": "port",
                         "sample": f"{args.steps} steps (rebuild every {args.nstlist}) of the full workload"},
        "e2e": {"value": value, "unit": "pairs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- GPU arm
def run_ours(args):
    import torch

    import paper_1506_00716_b200 as nbx
    from paper_1506_00716_b200 import _lib
    from paper_1506_00716_b200.kernels import flops_per_pair

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        return run_dd(args, world, rank, local)
    dist = None
    lib = _lib.load()
    system, table, occ = workload(args)
    params = nbx.NonbondedParams(**{k: getattr(make_params(args, table), k) for k in (
        "r_cut", "r_list", "lj_table", "coulomb_scale", "shift_potential", "elec", "epsilon_rf", "ewald_beta")})
    box = system.box
    dev = torch.device("cuda", local)
    pos_d = torch.from_numpy(np.array(system.positions)).to(dev)
    q_d = torch.from_numpy(np.array(system.charges)).to(dev)
    t_d = torch.from_numpy(np.array(system.lj_type)).to(dev)
    f_d = torch.empty((system.n, 3), dtype=torch.float64, device=dev)
    e_d = torch.zeros(2, dtype=torch.float64, device=dev)
    bad_d = torch.empty(2, dtype=torch.int64, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    st = {}

    def rebuild(pos, q, t, out):
        grid = nbx.build_cluster_grid(system, M, occ, positions=pos)
        st["grid"] = grid
        st["plist"] = nbx.prune_pair_list(nbx.build_pair_list(grid, box, R_LIST), grid.clustered_positions_device, box,
                                          r_inner=args.rinner)

    def step(k, pos, q, t, out):
        if k % args.nstlist == 0 or "plist" not in st:
            rebuild(pos, q, t, out)
        # energies on list steps (nstcalcenergy = nstlist), forces every step
        nbx.compute_nonbonded_device(st["plist"], st["grid"], pos, q, t, params, box,
                                     energy=(k % args.nstlist == 0), out=out, e_out=e_d, bad=bad_d)

    clocks = Clocks(local)
    # setup (not timed, not counted as warm-up steps): two full list cycles so
    # the stream-ordered memory pool holds two list generations (steady state)
    for k in range(2 * args.nstlist if args.nstlist <= 50 else 2):
        step(k, pos_d, q_d, t_d, f_d)
    for k in range(max(3, args.warmup)):
        step(k, pos_d, q_d, t_d, f_d)
    torch.cuda.synchronize()
    if int(bad_d[0].item()) != -1:
        raise RuntimeError("singular pair in the benchmark system")
    stats = nbx.interaction_stats(st["plist"], st["grid"], st["grid"].clustered_positions_device, box, R_CUT)
    n_within, n_admitted = stats.n_within_cutoff, stats.n_admitted
    # pairs the force kernel evaluates (the inner list's under dynamic pruning;
    # the positions are static, so the inner list stays valid every step)
    n_force = st["plist"].force_pairs(inner=True)

    # ---- device-resident timed region
    W = max(3, args.warmup)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    launches0 = lib.nbx_launch_count()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    wall0 = time.perf_counter()
    for i in range(args.steps):
        flush.zero_()
        ev[i][0].record()
        step(W + i, pos_d, q_d, t_d, f_d)
        ev[i][1].record()
    torch.cuda.synchronize()
    wall = time.perf_counter() - wall0
    launches = lib.nbx_launch_count() - launches0
    lib.nbx_timing_enable(0)
    lib.nbx_timing_query(None, None)
    # k_force duration: events around every launch of K eager (non-energy)
    # passes on the launching stream, the same list as the timed region
    lib.nbx_timing_enable(1)
    for _ in range(args.steps):
        flush.zero_()
        nbx.compute_nonbonded_device(st["plist"], st["grid"], pos_d, q_d, t_d, params, box, energy=False,
                                     out=f_d, e_out=e_d, bad=bad_d)
    torch.cuda.synchronize()
    lib.nbx_timing_enable(0)
    fk_ms, fk_n = (np.zeros(1), np.zeros(1, dtype=np.int64))
    _lib.check(lib.nbx_timing_query(_lib.ptr(fk_ms), _lib.ptr(fk_n)), "timing")
    clk = clocks.stop()
    t_ms = float(sum(a.elapsed_time(b) for a, b in ev))
    if os.environ.get("NBX_BENCH_DEBUG"):
        print("per-step ms:", [round(a.elapsed_time(b), 3) for a, b in ev], file=sys.stderr)
    if dist is not None:
        tt = torch.tensor([t_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_ms = float(tt.item())
    value = world * n_within * args.steps / (t_ms * 1e-3)

    # ---- end-to-end through the public API with host (pinned) buffers
    pos_h = torch.from_numpy(np.array(system.positions)).pin_memory()
    q_h = torch.from_numpy(np.array(system.charges)).pin_memory()
    t_h = torch.from_numpy(np.array(system.lj_type)).pin_memory()
    f_h = torch.empty((system.n, 3), dtype=torch.float64).pin_memory()
    e_h = torch.empty(2, dtype=torch.float64).pin_memory()
    pos_s = torch.empty_like(pos_d)
    q_s = torch.empty_like(q_d)
    t_s = torch.empty_like(t_d)
    st.clear()
    ev2 = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for i in range(W + args.steps):
        if i >= W:
            flush.zero_()
            ev2[i - W][0].record()
        pos_s.copy_(pos_h, non_blocking=True)
        q_s.copy_(q_h, non_blocking=True)
        t_s.copy_(t_h, non_blocking=True)
        step(i, pos_s, q_s, t_s, f_d)
        f_h.copy_(f_d, non_blocking=True)
        e_h.copy_(e_d, non_blocking=True)
        if i >= W:
            ev2[i - W][1].record()
    torch.cuda.synchronize()
    e2e_ms = float(sum(a.elapsed_time(b) for a, b in ev2))
    if dist is not None:
        tt = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_ms = float(tt.item())
    h2d = system.n * (24 + 8 + 8)
    d2h = system.n * 24 + 16

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
        "ms_per_step": t_ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "fp32 (pair math; fp64 energy + final force accumulation)",
        "data": "synthetic (seeded SPC-geometry water, BASELINE.md recipe)",
        "config": config(args, occ),
        "ns_per_day": args.steps / (t_ms * 1e-3) * DT_PS * 86.4,
        "pairs_per_step": {"within_rc": n_within, "admitted": n_admitted, "force_kernel": n_force,
                           "admitted_per_s": world * n_admitted * args.steps / (t_ms * 1e-3)},
        "e2e": {"value": world * n_within * args.steps / (e2e_ms * 1e-3), "unit": "pairs/s",
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "ms_per_step": e2e_ms / args.steps},
        "gpu_launches": int(launches),
        "roofline": {"bound": "fp32", "kernel": "k_force", "achieved": achieved, "peak": peak_tf,
                     "unit": "TFLOP/s", "frac": achieved / peak_tf, "traffic": traffic,
                     "kernel_ms": fk_avg_ms, "flops_per_pair": fpp, "pairs": "force_kernel (admitted pairs the kernel evaluates)",
                     "peak_note": f"nominal FP32: {n_sm} SMs x 128 lanes x 2 x {sm_max:.0f} MHz (sm_max_mhz of MEASURED_PEAKS.json)"},
        "clocks": clk,
        "wall_s_timed": wall,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        c = cpu_port_times(system, oracle_physics(params), occ, args.nstlist)
        per_step = c["force"] + (c["grid"] + c["search"] + c["prune"]) / args.nstlist
        line["cpu_baseline"] = {
            "value": n_within / per_step, "unit": "pairs/s", "cores": c["threads"], "kind": "port",
            "sample": (f"one rebuild (grid {c['grid']:.3f}s, O(n_c^2) search {c['search']:.3f}s, "
                       f"prune {c['prune']:.3f}s) + one force pass {c['force']:.3f}s, amortised over "
                       f"nstlist={args.nstlist}")}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def run_dd(args, world, rank, local):
    """N > 1: strong scaling of the same box over N GPUs with the slab
    decomposition (paper_1506_00716_b200/dd.py): per step NCCL halo exchange
    (coordinates in, forces back), local search every nstlist steps after an
    all-gather of home positions, energies all-reduced on energy steps."""
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
    dd = SlabDecomposition(box.lengths, world, rank, r_comm=R_LIST)
    dd.enable_native()
    p2p = dd.enable_p2p(system.n)  # per-step halo exchanges as NVLink peer stores (NBX_DD_P2P=0: NCCL)
    df = DomainForces(dd, system, params, M, occ, r_inner=args.rinner)
    pos_glob = torch.from_numpy(np.array(system.positions)).to(dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    lay = df.rebuild(pos_glob)

    def step(k, home_pos=None):
        nonlocal lay
        if k % args.nstlist == 0:
            cur = df.local_pos[:lay.n_home] if home_pos is None else home_pos
            glob = dd.allgather_home(lay.home, cur, system.n)
            lay = df.rebuild(glob)
        elif home_pos is not None:
            df.local_pos[:lay.n_home].copy_(home_pos)
        return df.forces(energy=(k % args.nstlist == 0))

    W = max(3, args.warmup)
    for k in range(2 * args.nstlist if args.nstlist <= 50 else 2):  # setup: memory pool steady state
        step(k)
    for k in range(W):
        step(k)
    torch.cuda.synchronize()
    st = nbx.interaction_stats(df.plist, df.grid, df.grid.clustered_positions_device, box, R_CUT)
    cnt = torch.tensor([st.n_within_cutoff, st.n_admitted], dtype=torch.int64, device=dev)
    dist.all_reduce(cnt)
    n_within, n_admitted = int(cnt[0].item()), int(cnt[1].item())
    n_force_rank = df.plist.force_pairs(inner=True)  # this rank's kernel work (inner list if any)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    clocks = Clocks(local)
    lib.nbx_timing_query(None, None)
    lib.nbx_timing_enable(1)
    launches0 = lib.nbx_launch_count()
    dist.barrier()
    torch.cuda.synchronize()
    for i in range(args.steps):
        flush.zero_()
        ev[i][0].record()
        step(W + i)
        ev[i][1].record()
    torch.cuda.synchronize()
    launches = lib.nbx_launch_count() - launches0
    lib.nbx_timing_enable(0)
    fk_ms, fk_n = np.zeros(1), np.zeros(1, dtype=np.int64)
    _lib.check(lib.nbx_timing_query(_lib.ptr(fk_ms), _lib.ptr(fk_n)), "timing")
    clk = clocks.stop()
    t = torch.tensor([sum(a.elapsed_time(b) for a, b in ev)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_ms = float(t.item())
    # e2e: home positions H2D from pinned host memory, home forces + energies D2H, every step
    home_h = df.local_pos[:lay.n_home].cpu().pin_memory()
    ev2 = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    bytes_io = torch.zeros(2, dtype=torch.int64, device=dev)
    for i in range(W + args.steps):
        if i >= W:
            flush.zero_()
            ev2[i - W][0].record()
        if home_h.shape[0] != lay.n_home:
            home_h = df.local_pos[:lay.n_home].cpu().pin_memory()
        hp = home_h.to(dev, non_blocking=True)
        f, e = step(W + args.steps + i, home_pos=hp)
        f_host = torch.empty(f.shape, dtype=f.dtype).pin_memory()
        f_host.copy_(f, non_blocking=True)
        e_host = e.to("cpu", non_blocking=True)
        if i >= W:
            ev2[i - W][1].record()
            bytes_io[0] += hp.numel() * 8
            bytes_io[1] += f.numel() * 8 + 16
    torch.cuda.synchronize()
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
        line = {
            "metric": "nonbonded pair-interactions/s (useful, r<=r_c)",
            "value": n_within * args.steps / (t_ms * 1e-3), "unit": "pairs/s", "n_gpus": world,
            "steps": args.steps, "warmup": W, "ms_per_step": t_ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None,
            "dtype": "fp32 (pair math; fp64 energy + final force accumulation)",
            "data": "synthetic (seeded SPC-geometry water, BASELINE.md recipe)",
            "config": config(args, occ, {"parallelism": f"slab DD x{world} (half-shell halo, r_comm=r_list, "
                                                         f"{'NVLink peer stores' if p2p else 'NCCL send/recv'})"}),
            "ns_per_day": args.steps / (t_ms * 1e-3) * DT_PS * 86.4,
            "pairs_per_step": {"within_rc": n_within, "admitted": n_admitted},
            "e2e": {"value": n_within * args.steps / (e2e_ms * 1e-3), "unit": "pairs/s",
                    "h2d_bytes_per_step": int(bytes_io[0].item()) // args.steps,
                    "d2h_bytes_per_step": int(bytes_io[1].item()) // args.steps, "ms_per_step": e2e_ms / args.steps},
            "gpu_launches": int(launches),
            "roofline": {"bound": "fp32", "kernel": "k_force (rank 0)", "achieved": achieved, "peak": peak_tf,
                         "unit": "TFLOP/s", "frac": achieved / peak_tf, "traffic": None, "kernel_ms": fk_avg_ms,
                         "flops_per_pair": flops_per_pair(params),
                         "pairs": "force_kernel of rank 0 (admitted pairs the kernel evaluates)"},
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    dist.barrier()
    dist.destroy_process_group()


def main():
    global R_LIST
    args = parse()
    R_LIST = args.rlist
    if args.rinner is None:
        args.rinner = min(R_CUT + 0.02, R_LIST)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
