"""Drop-in list rebuild at 96k: per-phase wall time with a sync after each phase, staging costs, cProfile."""
import sys, time; sys.path.insert(0, "/root/repo")
import numpy as np, torch, cProfile, pstats
import paper_1506_00716_b200 as nbx
from paper_1506_00716_b200.systems import spc_water, tuned_occupancy
from paper_1506_00716_b200 import _device as dv
s, table = spc_water(96000); box = s.box
occ = tuned_occupancy(96000, float(box.lengths[0]), 4)
q, t = np.array(s.charges), np.array(s.lj_type); p = np.array(s.positions)
def sync(): torch.cuda.synchronize(); return time.perf_counter()
acc = {}
for it in range(30):
    a = sync(); sysk = nbx.ParticleSystem(positions=p, velocities=s.velocities, masses=s.masses, charges=q, lj_type=t, box=box)
    b = sync(); g = nbx.build_cluster_grid(sysk, 4, occ)
    c = sync(); bl = nbx.build_pair_list(g, box, 1.1)
    d = sync(); cp = g.clustered_positions
    e = sync(); pl = nbx.prune_pair_list(bl, cp, box)
    f = sync()
    if it >= 10:
        for k, v in dict(system=b-a, grid=c-b, build=d-c, cpos=e-d, prune=f-e).items(): acc[k] = acc.get(k, 0) + v / 20
print({k: round(v*1e3, 3) for k, v in acc.items()})
cpos_t = torch.zeros(g.n_slots, 3, dtype=torch.float64, device="cuda")
def tm(fn, k=20):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(k): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / k * 1e3
print("stage_out 2.3MB", tm(lambda: dv.stage_out(cpos_t, "x")))
print("stage_out nocopy", tm(lambda: dv.stage_out(cpos_t, "y", copy=False)))
print("np.empty+copy 2.3MB", tm(lambda: np.empty((g.n_slots, 3)).__setitem__(slice(None), 1.0)))
print("stage_in positions", tm(lambda: dv.stage_in(p, torch.float64, "positions")))
pr = cProfile.Profile(); pr.enable()
for _ in range(20):
    sysk = nbx.ParticleSystem(positions=p, velocities=s.velocities, masses=s.masses, charges=q, lj_type=t, box=box)
    g = nbx.build_cluster_grid(sysk, 4, occ); bl = nbx.build_pair_list(g, box, 1.1)
    pl = nbx.prune_pair_list(bl, g.clustered_positions, box)
torch.cuda.synchronize()
pr.disable(); pstats.Stats(pr).sort_stats("tottime").print_stats(14)
