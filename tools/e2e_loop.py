"""The bench's drop-in e2e loop with per-step timings split into rebuild and
force-only steps (where the 1-2 ms/step of the drop-in path goes)."""
import sys, time; sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_1506_00716_b200 as nbx
from paper_1506_00716_b200.systems import spc_water, tuned_occupancy
import bench

s, table = spc_water(96000); box = s.box
occ = tuned_occupancy(96000, float(box.lengths[0]), 4)
params = nbx.NonbondedParams(r_cut=1.0, r_list=1.1, lj_table=table, shift_potential=True, elec="ewald",
                             ewald_beta=nbx.ewald_beta(1.0))
traj = bench.Trajectory(s)
lay = nbx.KernelLayout(4, 4)
q, t = np.array(s.charges), np.array(s.lj_type)
host = [traj.host(k) for k in range(60)]
de, rows = {}, []
for k in range(60):
    p = host[k]
    t0 = time.perf_counter()
    rb = "plist" not in de or k - de["build"] >= 10
    ph = {}
    if rb:
        a = time.perf_counter()
        sysk = nbx.ParticleSystem(positions=p, velocities=s.velocities, masses=s.masses, charges=q, lj_type=t, box=box)
        b = time.perf_counter(); g = nbx.build_cluster_grid(sysk, 4, occ)
        c = time.perf_counter(); bl = nbx.build_pair_list(g, box, 1.1)
        d = time.perf_counter(); cp = g.clustered_positions
        e = time.perf_counter(); pl = nbx.prune_pair_list(bl, cp, box)
        f = time.perf_counter()
        ph = dict(system=b - a, grid=c - b, build=d - c, cpos=e - d, prune=f - e)
        de.update(grid=g, plist=pl, build=k)
    a = time.perf_counter()
    nbx.compute_nonbonded_original(de["plist"], de["grid"], p, q, t, params, box, lay)
    ph["force"] = time.perf_counter() - a
    rows.append((rb, time.perf_counter() - t0, ph))
rows = rows[10:]
for rb in (True, False):
    sel = [r for r in rows if r[0] == rb]
    keys = sel[0][2].keys()
    print("rebuild" if rb else "force-only", len(sel), "steps, ms/step %.3f" % (1e3 * np.mean([r[1] for r in sel])),
          {k: round(1e3 * np.mean([r[2][k] for r in sel]), 3) for k in keys})
print("mean ms/step %.3f" % (1e3 * np.mean([r[1] for r in rows])))
