"""Host vs device time of the list step (grid + list + prune + first force
pass) at 96k, without a profiler: where the host keeps the GPU waiting.
    python tools/host_list_step.py [atoms]"""
import cProfile
import pstats
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1506_00716_b200 as nbx  # noqa: E402
from paper_1506_00716_b200.systems import spc_water, tuned_occupancy  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 96000
s, table = spc_water(n)
occ = tuned_occupancy(n, float(s.box.lengths[0]), 4)
params = nbx.NonbondedParams(r_cut=1.0, r_list=1.1, lj_table=table, shift_potential=True, elec="ewald",
                             ewald_beta=nbx.ewald_beta(1.0))
dev = torch.device("cuda", 0)
pos = torch.from_numpy(np.array(s.positions)).to(dev)
q = torch.from_numpy(np.array(s.charges)).to(dev)
t = torch.from_numpy(np.array(s.lj_type)).to(dev)
f = torch.empty_like(pos)


def phases():
    out = {}
    t0 = time.perf_counter()
    grid = nbx.build_cluster_grid(s, 4, occ, positions=pos)
    t1 = time.perf_counter()
    built = nbx.build_pair_list(grid, s.box, 1.1)
    t2 = time.perf_counter()
    pl = nbx.prune_pair_list(built, grid.clustered_positions_device, s.box)
    t3 = time.perf_counter()
    nbx.compute_nonbonded_device(pl, grid, pos, q, t, params, s.box, energy=False, out=f)
    t4 = time.perf_counter()
    out.update(grid=t1 - t0, build=t2 - t1, prune=t3 - t2, force=t4 - t3)
    return out, (grid, pl)


for _ in range(5):
    phases()
torch.cuda.synchronize()
hs = []
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(10):
    torch.cuda.synchronize()
    a.record()
    h0 = time.perf_counter()
    ph, keep = phases()
    h1 = time.perf_counter()
    b.record()
    torch.cuda.synchronize()
    hs.append((h1 - h0, a.elapsed_time(b) * 1e-3, ph))
h = np.median([x[0] for x in hs]) * 1e6
d = np.median([x[1] for x in hs]) * 1e6
print(f"list step + first force pass: host enqueue {h:.0f} us, device span {d:.0f} us")
for k in hs[0][2]:
    print(f"  host {k}: {np.median([x[2][k] for x in hs]) * 1e6:.0f} us")
pr = cProfile.Profile()
pr.enable()
for _ in range(10):
    phases()
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
