"""Wall time of the DD list-step bookkeeping: migrate (neighbour exchanges)
vs allgather_home + assign, per phase of migrate (torchrun, NCCL).
    torchrun --nproc-per-node N tools/dd_migrate_time.py [atoms]"""
import datetime
import os
import sys
import time
from pathlib import Path

import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
from paper_1506_00716_b200.dd import SlabDecomposition  # noqa: E402
from paper_1506_00716_b200.systems import spc_water  # noqa: E402

rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
dist.init_process_group("nccl", device_id=dev, timeout=datetime.timedelta(seconds=90))
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1500000
s, _ = spc_water(n)
traj = bench.Trajectory(s)
dd = SlabDecomposition(s.box.lengths, world, rank, r_comm=1.1)
dd.balance_counts(traj.host(0)[:, 0])
dd.enable_native()
lay = dd.assign(torch.from_numpy(traj.host(0)).to(dev))
pos = {k: torch.from_numpy(traj.host(k)).to(dev) for k in range(0, 80, 10)}


def t(fn):
    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    return r, 1e3 * (time.perf_counter() - t0)


for k in range(10, 80, 10):
    hp = pos[k].index_select(0, lay.home)
    (lay_m, _), tm = t(lambda: dd.migrate(lay.home, hp))
    _, ta = t(lambda: dd.assign(dd.allgather_home(lay.home, hp, s.n)) if getattr(dd, "home_counts", None) is not None
              else dd.assign(pos[k]))
    lay = dd.layout
    if rank == 0:
        print(f"N={world} k={k}: migrate {tm:.3f} ms, (allgather +) assign {ta:.3f} ms")
# phases of one migrate (torch profiler of rank 0)
hp = pos[70].index_select(0, lay.home)
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CPU, torch.profiler.ProfilerActivity.CUDA]) as prof:
    dd.migrate(lay.home, hp)
    torch.cuda.synchronize()
if rank == 0:
    print(prof.key_averages().table(sort_by="cpu_time_total", row_limit=18))
dist.destroy_process_group()
