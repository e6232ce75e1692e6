"""NVLink peer-store halo exchange vs NCCL send/recv (torchrun, N ranks):
forces bit-identical, per-step device time of force-only DD steps."""
import datetime
import os
import sys
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
dist.init_process_group("nccl", device_id=torch.device("cuda", local), timeout=datetime.timedelta(seconds=60))
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
df.rebuild(pos)


def run(tag):
    f, e = df.forces(energy=True)
    f0 = f.clone()
    e0 = e.clone()
    for _ in range(5):
        df.forces(energy=False)
    torch.cuda.synchronize()
    dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(50):
        df.forces(energy=False)
    b.record()
    torch.cuda.synchronize()
    t = torch.tensor([a.elapsed_time(b) / 50 * 1e3], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        print(f"N={world} {tag}: force-only DD step {t.item():.1f} us (max over ranks)")
    return f0, e0


fn, en = run("nccl (sequential)")
ok = dd.enable_p2p(s.n)
df.overlap = False
df.halo_first = False
fs, es = run("p2p sequential, three calls " + str(ok))
df.halo_first = True
fh, eh = run("p2p sequential, halo forces first (nbx_dd_force_seq) " + str(ok))
df.overlap = True
fp, ep = run("p2p overlapped (nbx_dd_force) " + str(ok))
same = (torch.equal(fn, fp) and torch.equal(en, ep) and torch.equal(fn, fs) and torch.equal(en, es)
        and torch.equal(fn, fh) and torch.equal(en, eh))
flag = torch.tensor([0 if same else 1], device=dev)
dist.all_reduce(flag)
err = dd.p2p_error()
if rank == 0:
    print(f"N={world} forces bit-identical on every rank: {int(flag.item()) == 0}; p2p wait timeouts: {err}")
dist.barrier()
dist.destroy_process_group()
