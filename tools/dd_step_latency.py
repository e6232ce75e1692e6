"""Host enqueue time vs device time of the per-step DD force pass (torchrun).

    torchrun --nproc-per-node N tools/dd_step_latency.py [atoms]
"""
import datetime
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1506_00716_b200 as nbx  # noqa: E402
from paper_1506_00716_b200.dd import DomainForces, SlabDecomposition  # noqa: E402
from paper_1506_00716_b200.systems import spc_water, tuned_occupancy  # noqa: E402

rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local), timeout=datetime.timedelta(seconds=90))
n = int(sys.argv[1]) if len(sys.argv) > 1 else 96000
s, table = spc_water(n)
occ = tuned_occupancy(n, float(s.box.lengths[0]), 4)
params = nbx.NonbondedParams(r_cut=1.0, r_list=1.1, lj_table=table, shift_potential=True, elec="ewald",
                             ewald_beta=nbx.ewald_beta(1.0))
dev = torch.device("cuda", local)
pos = torch.from_numpy(np.array(s.positions)).to(dev)
dd = SlabDecomposition(s.box.lengths, world, rank, r_comm=1.1)
dd.enable_native()
df = DomainForces(dd, s, params, 4, occ)
lay = df.rebuild(pos)
for _ in range(5):
    df.forces(energy=True)
    df.forces(energy=False)
K = 50
for energy in (False, True):
    for rep in range(3):
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        h0 = time.perf_counter()
        for _ in range(K):
            df.forces(energy=energy)
        h1 = time.perf_counter()
        e1.record()
        torch.cuda.synchronize()
        h2 = time.perf_counter()
        if rank == 0:
            print(f"N={world} energy={energy} rep {rep}: host enqueue {1e3 * (h1 - h0) / K:.3f} ms/step | "
                  f"device {e0.elapsed_time(e1) / K:.3f} ms/step | wall {1e3 * (h2 - h0) / K:.3f}", flush=True)
# device time of one force pass alone (no exchange)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(K):
    nbx.compute_nonbonded_device(df.plist, df.grid, df.local_pos, df.q, df.t, params, s.box, energy=False,
                                 out=df.f, e_out=df.e, bad=df.bad)
e1.record()
torch.cuda.synchronize()
if rank == 0:
    print(f"N={world} local force only: {e0.elapsed_time(e1) / K:.3f} ms/step, home {lay.n_home} "
          f"halo {lay.n_local - lay.n_home}", flush=True)
dist.destroy_process_group()
