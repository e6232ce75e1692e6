"""Device-resident MD (engine.run_md) throughput: the oxygen sites of the
SPC water box as an LJ fluid (charges off -- the reference's SPC water has no
intramolecular exclusions or constraints and collapses within a few steps,
SURVEY §0.3), 300 K, dt = 2 fs, nstlist 10 with the drift guard.

    python tools/md_bench.py [--atoms 96000] [--steps 500] [--nstlist 10] [--rlist 1.1] [--json]

--nstlist/--rlist give BASELINE config 5 (Verlet-buffer sweep nstlist 10/20/40
with r_list 1.1/1.15/1.2): how many rebuilds the drift guard forces and what
the buffer costs per step (tools/nstlist_sweep.sh).
"""
import argparse
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1506_00716_b200 as nbx  # noqa: E402
from paper_1506_00716_b200.systems import spc_water, tuned_occupancy  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--atoms", type=int, default=96000)
ap.add_argument("--steps", type=int, default=500)
ap.add_argument("--nstlist", type=int, default=10)
ap.add_argument("--rlist", type=float, default=1.1)
ap.add_argument("--json", action="store_true", help="print one JSON summary line last")
ap.add_argument("--rinner", type=float, default=0.0, help="dynamic pruning inner radius (0 = off)")
ap.add_argument("--prune-interval", type=int, default=0, help="rolling prune every N steps (0 = off)")
a = ap.parse_args()
w, table = spc_water(a.atoms, temperature=300.0)
o = np.arange(0, w.n, 3)
s = nbx.ParticleSystem(positions=w.positions[o], velocities=w.velocities[o], masses=w.masses[o],
                       charges=np.zeros(o.size), lj_type=np.zeros(o.size, dtype=np.int64), box=w.box)
params = nbx.NonbondedParams(r_cut=1.0, r_list=a.rlist, lj_table=table[:1, :1], shift_potential=True)
layout = nbx.KernelLayout(4, 4)
occ = tuned_occupancy(s.n, float(s.box.lengths[0]), 4)
pol = nbx.ListPolicy(rebuild_interval=a.nstlist, r_inner=a.rinner, prune_interval=a.prune_interval)
nbx.run_md(s, params, layout, 0.002, 20, policy=pol, report_interval=10, target_occupancy=occ)  # warm-up
torch.cuda.synchronize()
t0 = time.perf_counter()
res = nbx.run_md(s, params, layout, 0.002, a.steps, policy=pol, report_interval=100, target_occupancy=occ)
torch.cuda.synchronize()
wall = time.perf_counter() - t0
ms = 1e3 * wall / a.steps
print(f"LJ fluid {s.n} atoms: {a.steps} steps in {wall:.3f} s = {ms:.3f} ms/step, "
      f"{0.002 * a.steps / wall * 86.4:.1f} ns/day (wall, incl. setup + reports) | rebuilds {res.state.n_rebuilds} "
      f"(drift {res.state.n_drift_rebuilds}) | T {res.temperature[0]:.1f} -> {res.temperature[-1]:.1f} K | "
      f"energy drift rel {res.energy_drift()[1]:.2e}")
for k, (cnt, t) in res.timing.sections.items():
    print(f"  {k:10s} {cnt:6d} calls {1e3 * t:9.2f} ms")
if a.json:
    import json
    print(json.dumps({"tool": "md_bench", "n_atoms": int(s.n), "nstlist": a.nstlist, "r_list_nm": a.rlist,
                      "steps": a.steps, "r_inner_nm": a.rinner, "prune_interval": a.prune_interval, "ms_per_step": ms, "ns_per_day": 0.002 * a.steps / wall * 86.4,
                      "rebuilds": int(res.state.n_rebuilds), "drift_rebuilds": int(res.state.n_drift_rebuilds),
                      "energy_drift_rel": float(res.energy_drift()[1])}))
