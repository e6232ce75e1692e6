"""Multi-GPU check of the list step by migration (torchrun, NCCL): after the
bench trajectory moves the atoms, DomainForces.rebuild_local (neighbour
exchanges only) gives every rank the same layout, local positions and
bit-identical forces / energies as rebuild() from the all-gathered positions.
    torchrun --nproc-per-node N tools/dd_migrate_check.py [atoms]"""
import datetime
import os
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_1506_00716_b200.dd import DomainForces, SlabDecomposition  # noqa: E402
from paper_1506_00716_b200.systems import spc_water, tuned_occupancy  # noqa: E402
import paper_1506_00716_b200 as nbx  # noqa: E402

rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
dist.init_process_group("nccl", device_id=dev, timeout=datetime.timedelta(seconds=90))
n = int(sys.argv[1]) if len(sys.argv) > 1 else 96000
s, table = spc_water(n)
occ = tuned_occupancy(n, float(s.box.lengths[0]), 4)
params = nbx.NonbondedParams(r_cut=1.0, r_list=1.1, lj_table=table, shift_potential=True, elec="ewald",
                             ewald_beta=nbx.ewald_beta(1.0))
traj = bench.Trajectory(s)
ok = True
for p2p in (False, True):
    dd = SlabDecomposition(s.box.lengths, world, rank, r_comm=1.1)
    dd.balance_counts(traj.host(0)[:, 0])
    dd.enable_native()
    if p2p:
        dd.enable_p2p(s.n)
    df = DomainForces(dd, s, params, 4, occ)
    lay = df.rebuild(torch.from_numpy(traj.host(0)).to(dev))
    for k in (10, 20, 30):
        glob = torch.from_numpy(traj.host(k)).to(dev)
        home_pos = glob.index_select(0, lay.home)
        lay_m = df.rebuild_local(lay.home, home_pos)
        f_m, e_m = df.forces(energy=True)
        f_m, e_m = f_m.clone(), e_m.clone()
        ref = DomainForces(dd, s, params, 4, occ)
        lay_r = ref.rebuild(glob)
        f_r, e_r = ref.forces(energy=True)
        same = all(torch.equal(getattr(lay_m, a), getattr(lay_r, a)) for a in ("home", "halo", "send_local"))
        same &= torch.equal(df.local_pos, ref.local_pos) and torch.equal(f_m, f_r) and torch.equal(e_m, e_r)
        ok &= bool(same)
        # (ref.rebuild re-set the shared exchange layout to the same sets)
        lay = lay_m
    dd.check_p2p()
    dd.close()
t = torch.tensor([1 if ok else 0], device=dev)
dist.all_reduce(t, op=dist.ReduceOp.MIN)
if rank == 0:
    print("MIGRATE PARITY", "OK" if int(t.item()) == 1 else "FAILED")
dist.destroy_process_group()
