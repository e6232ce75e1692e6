"""Drop-in (numpy) API cost breakdown at 96k: compute_nonbonded_original vs its staging, device force and
read-back pieces; list rebuild pieces (ParticleSystem, grid, build, clustered_positions, prune)."""
import sys, time; sys.path.insert(0, "/root/repo")
import numpy as np, torch, cProfile, pstats
import paper_1506_00716_b200 as nbx
from paper_1506_00716_b200.systems import spc_water, tuned_occupancy
s, table = spc_water(96000); occ = tuned_occupancy(96000, float(s.box.lengths[0]), 4)
params = nbx.NonbondedParams(r_cut=1.0, r_list=1.1, lj_table=table, shift_potential=True, elec="ewald", ewald_beta=nbx.ewald_beta(1.0))
grid = nbx.build_cluster_grid(s, 4, occ); pl = nbx.prune_pair_list(nbx.build_pair_list(grid, s.box, 1.1), grid.clustered_positions, s.box)
lay = nbx.KernelLayout(4, 4)
pos = np.array(s.positions); q = np.array(s.charges); t = np.array(s.lj_type)
for _ in range(5): nbx.compute_nonbonded_original(pl, grid, pos, q, t, params, s.box, lay)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(20): nbx.compute_nonbonded_original(pl, grid, pos, q, t, params, s.box, lay)
print("force call ms", (time.perf_counter()-t0)/20*1e3)
t0 = time.perf_counter()
for _ in range(5):
    sysk = nbx.ParticleSystem(positions=pos, velocities=s.velocities, masses=s.masses, charges=q, lj_type=t, box=s.box)
    g = nbx.build_cluster_grid(sysk, 4, occ); p2 = nbx.prune_pair_list(nbx.build_pair_list(g, s.box, 1.1), g.clustered_positions, s.box)
torch.cuda.synchronize()
print("rebuild ms", (time.perf_counter()-t0)/5*1e3)
pr = cProfile.Profile(); pr.enable()
for _ in range(20): nbx.compute_nonbonded_original(pl, grid, pos, q, t, params, s.box, lay)
pr.disable(); pstats.Stats(pr).sort_stats("tottime").print_stats(10)

import time as _t
from paper_1506_00716_b200 import _device as dv
def tm(fn, k=20):
    torch.cuda.synchronize(); t0 = _t.perf_counter()
    for _ in range(k): r = fn()
    torch.cuda.synchronize(); return (_t.perf_counter() - t0) / k * 1e3
print("stage_in positions ms", tm(lambda: dv.stage_in(pos, torch.float64, "positions")))
print("stage_in charges (cached) ms", tm(lambda: dv.stage_in(s.charges, torch.float64, "charges")))
pt = dv.stage_in(pos, torch.float64, "positions")
qt = dv.stage_in(q, torch.float64, "charges"); tt = dv.stage_in(t, torch.int64, "lj_types")
print("device force (energy) ms", tm(lambda: nbx.compute_nonbonded_device(pl, grid, pt, qt, tt, params, s.box)))
f, e, b = nbx.compute_nonbonded_device(pl, grid, pt, qt, tt, params, s.box)
print("stage_out forces ms", tm(lambda: dv.stage_out(f, "forces")))
print("np.copyto 2.3MB into pinned ms", tm(lambda: np.copyto(dv._pinned["positions"].numpy(), pos.reshape(-1))))

def manual():
    pt = dv.stage_in(pos, torch.float64, "positions")
    qt = dv.stage_in(q, torch.float64, "charges"); tt = dv.stage_in(t, torch.int64, "lj_types")
    f, e, b = nbx.compute_nonbonded_device(pl, grid, pt, qt, tt, params, s.box)
    return dv.stage_out(f, "forces"), dv.stage_out(torch.cat([e, b.to(torch.float64)]), "energies")
print("manual sequence ms", tm(manual))
print("compute_nonbonded_original ms", tm(lambda: nbx.compute_nonbonded_original(pl, grid, pos, q, t, params, s.box, lay)))
import paper_1506_00716_b200.kernels as K
print("_check_shapes ms", tm(lambda: K._check_shapes(pl, grid, lay, pos.shape[0]), 200))
f, e, b = nbx.compute_nonbonded_device(pl, grid, pt, qt, tt, params, s.box)
print("bad", b.cpu().numpy(), "finite", bool(torch.isfinite(f).all()))
def rb():
    sysk = nbx.ParticleSystem(positions=pos, velocities=s.velocities, masses=s.masses, charges=q, lj_type=t, box=s.box)
    g = nbx.build_cluster_grid(sysk, 4, occ)
    return nbx.prune_pair_list(nbx.build_pair_list(g, s.box, 1.1), g.clustered_positions, s.box)
def ps():
    return nbx.ParticleSystem(positions=pos, velocities=s.velocities, masses=s.masses, charges=q, lj_type=t, box=s.box)
print("ParticleSystem ms", tm(ps))
sysk = ps()
print("grid ms", tm(lambda: nbx.build_cluster_grid(sysk, 4, occ)))
g = nbx.build_cluster_grid(sysk, 4, occ)
print("build ms", tm(lambda: nbx.build_pair_list(g, s.box, 1.1)))
bl = nbx.build_pair_list(g, s.box, 1.1)
print("clustered_positions ms", tm(lambda: nbx.build_cluster_grid(sysk, 4, occ).clustered_positions, 5))
print("prune (host cpos) ms", tm(lambda: nbx.prune_pair_list(bl, g.clustered_positions, s.box)))
