"""Long rigid-SPC MD run on the bench box (96k atoms, LJ + Ewald real space,
SETTLE + RATTLE, exclusions, NVE velocity Verlet at 2 fs): the bench's
relaxation to 300 K, then N steps (default 10^4) with energies every 100.
Writes gpurun_out/md_long.json (energy / temperature series, constraint
error at the end, list rebuilds, ns/day).
    python tools/md_long.py [--atoms 96000] [--steps 10000]"""
import argparse
import dataclasses
import json
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
ap.add_argument("--steps", type=int, default=10000)
ap.add_argument("--report", type=int, default=100)
a = ap.parse_args()
system, table = spc_water(a.atoms, seed=2024, temperature=300.0)
occ = tuned_occupancy(a.atoms, float(system.box.lengths[0]), 4)
params = nbx.NonbondedParams(r_cut=1.0, r_list=1.1, lj_table=table, shift_potential=True, elec="ewald",
                             ewald_beta=nbx.ewald_beta(1.0))
water = nbx.RigidWater()
layout = nbx.KernelLayout(4, 4)
dt = 0.002
for _ in range(5):  # the bench's relaxation: 5 x 20 steps, rescaled to 300 K between them
    res = nbx.run_md(system, params, layout, dt, 20, report_interval=20, target_occupancy=occ, constraints=water)
    v = res.state.system.velocities * np.sqrt(300.0 / max(float(res.temperature[-1]), 1.0))
    system = dataclasses.replace(res.state.system, velocities=v)
torch.cuda.synchronize()
t0 = time.perf_counter()
res = nbx.run_md(system, params, layout, dt, a.steps, report_interval=a.report, target_occupancy=occ,
                 constraints=water)
torch.cuda.synchronize()
wall = time.perf_counter() - t0 - res.timing.total("setup")
e = res.e_total
ke = float(np.mean(res.e_kinetic))
x = np.asarray(res.state.system.positions).reshape(-1, 3, 3)
L = np.asarray(system.box.lengths)


def bond(a, b):
    d = x[:, a] - x[:, b]
    d -= L * np.round(d / L)
    return np.linalg.norm(d, axis=1)


oh = float(max(np.abs(bond(0, 1) - water.d_oh).max(), np.abs(bond(0, 2) - water.d_oh).max()) / water.d_oh)
hh = float(np.abs(bond(1, 2) - water.d_hh).max() / water.d_hh)
drift_fit = np.polyfit(res.steps * dt, e, 1)[0] if len(e) > 2 else 0.0
out = {
    "system": f"{a.atoms // 3} rigid SPC waters, LJ + Ewald real space (erfc), r_c 1.0, r_list 1.1, nstlist 10",
    "steps": a.steps, "dt_ps": dt, "simulated_ps": a.steps * dt,
    "ns_per_day": a.steps / wall * dt * 86.4, "ms_per_step": 1e3 * wall / a.steps,
    "rebuilds": res.state.n_rebuilds, "drift_rebuilds": res.state.n_drift_rebuilds,
    "temperature_K": {"first": float(res.temperature[0]), "last": float(res.temperature[-1]),
                      "mean": float(np.mean(res.temperature)), "min": float(np.min(res.temperature)),
                      "max": float(np.max(res.temperature))},
    "energy_kj_mol": {"first": float(e[0]), "last": float(e[-1]), "mean_ke": ke,
                      "max_excursion_over_ke": float(np.abs(e - e[0]).max() / ke),
                      "linear_drift_kj_mol_per_ps_per_atom": float(drift_fit / a.atoms)},
    "constraints_max_rel_error": {"oh": oh, "hh": hh},
    "finite": bool(np.isfinite(e).all()),
    "series": {"step": res.steps.tolist(), "e_total": [round(float(x), 3) for x in e],
               "temperature": [round(float(x), 2) for x in res.temperature]},
}
Path("gpurun_out").mkdir(exist_ok=True)
Path("gpurun_out/md_long.json").write_text(json.dumps(out, indent=1))
print(json.dumps({k: v for k, v in out.items() if k != "series"}, indent=1))
