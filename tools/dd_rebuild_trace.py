"""Kernel timeline of one DD list step (all-gather + assign + local list
step + first force pass) on rank 0 (torchrun): GPU busy vs idle and the
largest host gaps.   torchrun --nproc-per-node N tools/dd_rebuild_trace.py [atoms]"""
import datetime
import json
import os
import sys
from collections import defaultdict
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
pos = {k: torch.from_numpy(traj.host(k)).to(dev) for k in range(0, 60, 10)}
lay = df.rebuild(pos[0])


def list_step(k):
    global lay
    hp = pos[k].index_select(0, lay.home)
    lay = df.rebuild(dd.allgather_home(lay.home, hp, s.n))
    df.forces(energy=True)


for k in (10, 20, 30):
    list_step(k)
torch.cuda.synchronize()
dist.barrier()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CPU,
                                        torch.profiler.ProfilerActivity.CUDA]) as prof:
    list_step(40)
    torch.cuda.synchronize()
dist.barrier()
if rank == 0:
    out = Path("gpurun_out")
    out.mkdir(exist_ok=True)
    prof.export_chrome_trace(str(out / "dd_rebuild_trace.json"))
    ev = json.load(open(out / "dd_rebuild_trace.json"))["traceEvents"]
    kern = sorted((e["ts"], e["ts"] + e.get("dur", 0), e["name"]) for e in ev
                  if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset"))
    span = kern[-1][1] - kern[0][0]
    busy, end, gaps = 0.0, kern[0][0], []
    for t0, t1, name in kern:
        if t0 > end:
            gaps.append((t0 - end, name))
        busy += max(0.0, t1 - max(t0, end))
        end = max(end, t1)
    print(f"N={world} rank 0 list step: span {span:.0f} us, GPU busy {busy:.0f}, idle {span - busy:.0f}, "
          f"{len(kern)} device activities")
    tot = defaultdict(lambda: [0, 0.0])
    for t0, t1, name in kern:
        tot[name.split("(")[0][:60]][0] += 1
        tot[name.split("(")[0][:60]][1] += t1 - t0
    for k, (c, d) in sorted(tot.items(), key=lambda x: -x[1][1])[:16]:
        print(f"   {c:3d} {d:8.1f} us  {k}")
    print("largest gaps:", ", ".join(f"{g:.0f}us<{nm.split('(')[0][:28]}" for g, nm in sorted(gaps, reverse=True)[:12]))
dd.close()
dist.destroy_process_group()
