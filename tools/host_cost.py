"""Host cost (µs per call, no device sync) of the force-step API layers."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1506_00716_b200 as nbx  # noqa: E402
from paper_1506_00716_b200 import _device, _lib  # noqa: E402
from paper_1506_00716_b200.kernels import _params_struct  # noqa: E402
from paper_1506_00716_b200.systems import spc_water, tuned_occupancy  # noqa: E402

s, table = spc_water(3000)
occ = tuned_occupancy(3000, float(s.box.lengths[0]), 4)
params = nbx.NonbondedParams(r_cut=1.0, r_list=1.1, lj_table=table, shift_potential=True, elec="ewald",
                             ewald_beta=nbx.ewald_beta(1.0))
dev = torch.device("cuda", 0)
pos = torch.from_numpy(np.array(s.positions)).to(dev)
q = torch.from_numpy(np.array(s.charges)).to(dev)
t = torch.from_numpy(np.array(s.lj_type)).to(dev)
out = torch.empty((s.n, 3), dtype=torch.float64, device=dev)
e = torch.zeros(2, dtype=torch.float64, device=dev)
bad = torch.empty(2, dtype=torch.int64, device=dev)
grid = nbx.build_cluster_grid(s, 4, occ, positions=pos)
pl = nbx.prune_pair_list(nbx.build_pair_list(grid, s.box, 1.1), grid.clustered_positions_device, s.box)


def bench(name, fn, n=2000):
    for _ in range(50):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    dt = (time.perf_counter() - t0) / n
    torch.cuda.synchronize()
    print(f"{name:40s} {1e6 * dt:7.2f} us")


bench("compute_nonbonded_device", lambda: nbx.compute_nonbonded_device(pl, grid, pos, q, t, params, s.box,
                                                                       energy=False, out=out, e_out=e, bad=bad))
bench("  _params_struct", lambda: _params_struct(params))
bench("  require_cuda", _device.require_cuda)
bench("  stream()", _device.stream)
bench("  box3", lambda: _lib.box3(s.box.lengths))
bench("  ptr x3", lambda: (_lib.ptr(pos), _lib.ptr(q), _lib.ptr(t)))
