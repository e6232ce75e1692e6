"""Host-side (Python + C API) cost of one list rebuild + force pass, cProfile."""
import cProfile
import pstats
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1506_00716_b200 as nbx  # noqa: E402
from paper_1506_00716_b200.systems import spc_water, tuned_occupancy  # noqa: E402

s, table = spc_water(96000)
occ = tuned_occupancy(96000, float(s.box.lengths[0]), 4)
params = nbx.NonbondedParams(r_cut=1.0, r_list=1.1, lj_table=table, shift_potential=True, elec="ewald",
                             ewald_beta=nbx.ewald_beta(1.0))
dev = torch.device("cuda", 0)
pos = torch.from_numpy(np.array(s.positions)).to(dev)
q = torch.from_numpy(np.array(s.charges)).to(dev)
t = torch.from_numpy(np.array(s.lj_type)).to(dev)
out = torch.empty((s.n, 3), dtype=torch.float64, device=dev)
e = torch.zeros(2, dtype=torch.float64, device=dev)
bad = torch.empty(2, dtype=torch.int64, device=dev)


def cycle():
    grid = nbx.build_cluster_grid(s, 4, occ, positions=pos)
    pl = nbx.prune_pair_list(nbx.build_pair_list(grid, s.box, 1.1), grid.clustered_positions_device, s.box)
    nbx.compute_nonbonded_device(pl, grid, pos, q, t, params, s.box, energy=True, out=out, e_out=e, bad=bad)
    for _ in range(9):
        nbx.compute_nonbonded_device(pl, grid, pos, q, t, params, s.box, energy=False, out=out, e_out=e, bad=bad)
    torch.cuda.synchronize()


for _ in range(3):
    cycle()
pr = cProfile.Profile()
pr.enable()
for _ in range(5):
    cycle()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
