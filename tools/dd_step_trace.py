"""Kernel timeline of force-only DD steps on rank 0 (torchrun, N ranks):
device time per kernel (incl. the peer-exchange put / take kernels) and the
GPU idle time of a step.   torchrun --nproc-per-node N tools/dd_step_trace.py [atoms]"""
import datetime
import json
import os
import sys
from collections import defaultdict
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
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1500000
s, table = spc_water(n)
occ = tuned_occupancy(n, float(s.box.lengths[0]), 4)
params = nbx.NonbondedParams(r_cut=1.0, r_list=1.1, lj_table=table, shift_potential=True, elec="ewald",
                             ewald_beta=nbx.ewald_beta(1.0))
dev = torch.device("cuda", local)
pos = torch.from_numpy(np.array(s.positions)).to(dev)
dd = SlabDecomposition(s.box.lengths, world, rank, r_comm=1.1)
dd.enable_native()
dd.enable_p2p(s.n)
df = DomainForces(dd, s, params, 4, occ)
df.rebuild(pos)
for _ in range(5):
    df.forces(energy=False)
torch.cuda.synchronize()
dist.barrier()
K = 10
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    for _ in range(K):
        df.forces(energy=False)
    torch.cuda.synchronize()
dist.barrier()
out = Path("gpurun_out")
out.mkdir(exist_ok=True)
prof.export_chrome_trace(str(out / f"dd_step_trace_r{rank}.json"))
ev = json.load(open(out / f"dd_step_trace_r{rank}.json"))["traceEvents"]
kern = sorted((e["ts"], e["ts"] + e.get("dur", 0), e["name"]) for e in ev
              if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset"))
span = kern[-1][1] - kern[0][0]
busy, end = 0.0, kern[0][0]
for t0, t1, _ in kern:
    busy += max(0.0, t1 - max(t0, end))
    end = max(end, t1)
tot = defaultdict(lambda: [0, 0.0])
ntake = 0
for t0, t1, name in kern:
    key = name.split("(")[0][:60]
    if "k_p2p_take" in key:  # 1st take of a step: halo positions in; 2nd: halo forces back
        key += " (positions)" if ntake % 2 == 0 else " (forces)"
        ntake += 1
    tot[key][0] += 1
    tot[key][1] += t1 - t0
lines = [f"N={world} rank {rank}: {K} force steps, span {span / K:.1f} us/step, busy {busy / K:.1f}, "
         f"idle {(span - busy) / K:.1f}, home {df.dd.layout.n_home} local {df.dd.layout.n_local}"]
for k, (c, d) in sorted(tot.items(), key=lambda x: -x[1][1]):
    lines.append(f"   {c // K:3d}x {d / K:8.1f} us/step  {k}")
allv = [None] * world
dist.all_gather_object(allv, "\n".join(lines))
if rank == 0:
    print("\n".join(allv))
dist.destroy_process_group()
