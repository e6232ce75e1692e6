"""Device time of DD force-only steps with and without each halo exchange
(positions in / forces back), to size what overlapping them could gain
(torchrun).   torchrun --nproc-per-node N tools/dd_exchange_cost.py [atoms]"""
import datetime
import os
import sys
from pathlib import Path

import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_1506_00716_b200 as nbx  # noqa: E402
from paper_1506_00716_b200.dd import DomainForces, SlabDecomposition  # noqa: E402
from paper_1506_00716_b200.systems import spc_water, tuned_occupancy  # noqa: E402

rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
dist.init_process_group("nccl", device_id=dev, timeout=datetime.timedelta(seconds=90))
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1500000
s, table = spc_water(n)
occ = tuned_occupancy(n, float(s.box.lengths[0]), 4)
params = nbx.NonbondedParams(r_cut=1.0, r_list=1.1, lj_table=table, shift_potential=True, elec="ewald",
                             ewald_beta=nbx.ewald_beta(1.0))
traj = bench.Trajectory(s)
dd = SlabDecomposition(s.box.lengths, world, rank, r_comm=1.1)
dd.balance_counts(traj.host(0)[:, 0])
dd.enable_native()
dd.enable_p2p(s.n)
df = DomainForces(dd, s, params, 4, occ)
df.rebuild(torch.from_numpy(traj.host(0)).to(dev))
real_x, real_f = dd.exchange_positions, dd.reduce_halo_forces


def timed(label, k=30):
    for _ in range(5):
        df.forces(energy=False)
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(k):
        df.forces(energy=False)
    e1.record()
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / k * 1e3], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(f"N={world} {label}: {t.item():.1f} us per force step (max over ranks)")


timed("both exchanges")
dd.reduce_halo_forces = lambda f: f[:dd.layout.n_home]
timed("positions only")
dd.exchange_positions = lambda x: None
timed("no exchange")
dd.exchange_positions, dd.reduce_halo_forces = real_x, real_f
timed("both exchanges (again)")
dd.close()
dist.destroy_process_group()
