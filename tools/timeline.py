"""Kernel timeline (torch.profiler / CUPTI) of one rebuild step and one force
step of the default bench workload: start offsets, durations and the idle gaps
between kernels.   python tools/timeline.py [--atoms 96000]"""
import argparse
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1506_00716_b200 as nbx  # noqa: E402
from paper_1506_00716_b200.systems import spc_water, tuned_occupancy  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--atoms", type=int, default=96000)
a = ap.parse_args()
s, table = spc_water(a.atoms)
occ = tuned_occupancy(a.atoms, float(s.box.lengths[0]), 4)
params = nbx.NonbondedParams(r_cut=1.0, r_list=1.1, lj_table=table, shift_potential=True, elec="ewald",
                             ewald_beta=nbx.ewald_beta(1.0))
dev = torch.device("cuda", 0)
pos = torch.from_numpy(np.array(s.positions)).to(dev)
q = torch.from_numpy(np.array(s.charges)).to(dev)
t = torch.from_numpy(np.array(s.lj_type)).to(dev)
out = torch.empty((s.n, 3), dtype=torch.float64, device=dev)
e = torch.zeros(2, dtype=torch.float64, device=dev)
bad = torch.empty(2, dtype=torch.int64, device=dev)


def rebuild_step():
    grid = nbx.build_cluster_grid(s, 4, occ, positions=pos)
    pl = nbx.prune_pair_list(nbx.build_pair_list(grid, s.box, 1.1), grid.clustered_positions_device, s.box)
    nbx.compute_nonbonded_device(pl, grid, pos, q, t, params, s.box, energy=True, out=out, e_out=e, bad=bad)
    return grid, pl


for _ in range(3):
    grid, pl = rebuild_step()
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    grid, pl = rebuild_step()
    nbx.compute_nonbonded_device(pl, grid, pos, q, t, params, s.box, energy=False, out=out, e_out=e, bad=bad)
    torch.cuda.synchronize()
ev = [x for x in prof.events() if x.device_type == torch.autograd.DeviceType.CUDA]
ev.sort(key=lambda x: x.time_range.start)
t0 = ev[0].time_range.start
prev = t0
busy = 0.0
for x in ev:
    st, en = x.time_range.start, x.time_range.end
    gap = st - prev
    busy += en - st
    print(f"{st - t0:9.1f} us  gap {gap:7.1f}  dur {en - st:8.1f}  {x.name[:90]}")
    prev = max(prev, en)
print(f"span {prev - t0:.1f} us, kernel busy {busy:.1f} us")

# host-side enqueue cost of each phase (no syncs inside)
import time  # noqa: E402

for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    grid = nbx.build_cluster_grid(s, 4, occ, positions=pos)
    t1 = time.perf_counter()
    bl = nbx.build_pair_list(grid, s.box, 1.1)
    t2 = time.perf_counter()
    pl = nbx.prune_pair_list(bl, grid.clustered_positions_device, s.box)
    t3 = time.perf_counter()
    nbx.compute_nonbonded_device(pl, grid, pos, q, t, params, s.box, energy=True, out=out, e_out=e, bad=bad)
    t4 = time.perf_counter()
    nbx.compute_nonbonded_device(pl, grid, pos, q, t, params, s.box, energy=False, out=out, e_out=e, bad=bad)
    t5 = time.perf_counter()
    torch.cuda.synchronize()
    t6 = time.perf_counter()
    print(f"host us: grid {1e6*(t1-t0):.0f} build {1e6*(t2-t1):.0f} prune {1e6*(t3-t2):.0f} "
          f"force1 {1e6*(t4-t3):.0f} force {1e6*(t5-t4):.0f} drain {1e6*(t6-t5):.0f}")
