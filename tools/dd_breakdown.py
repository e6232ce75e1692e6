"""Per-phase wall time of a DD rebuild + force pass (torchrun, N ranks)."""
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
df.forces(energy=True)


def t(fn):
    torch.cuda.synchronize()
    dist.barrier()
    t0 = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    return r, 1e3 * (time.perf_counter() - t0)


def rebuild_phases(glob):
    """DomainForces.rebuild split into its phases (same calls)."""
    from paper_1506_00716_b200 import build_cluster_grid, build_pair_list, prune_pair_list
    from paper_1506_00716_b200.dd import _Domain, local_occupancy

    out = {}
    lay, out["assign"] = t(lambda: dd.assign(glob))
    ids = lay.local_ids

    def gather():
        df.local_pos = glob.index_select(0, ids).contiguous()
        df.q = df.q_all.index_select(0, ids)
        df.t = df.t_all.index_select(0, ids)
        h = torch.zeros(lay.n_local, dtype=torch.uint8, device=dev)
        h[lay.n_home:] = 1
        df.halo = h
    _, out["gather"] = t(gather)
    o = occ
    if world > 1:
        o = local_occupancy(occ, lay.n_local, s.n, s.box.lengths, float(np.diff(dd.boundaries).max()), dd.r_comm)
    grid, out["grid"] = t(lambda: build_cluster_grid(_Domain(lay.n_local, s.box), 4, o, positions=df.local_pos))
    built, out["search"] = t(lambda: build_pair_list(grid, s.box, 1.1, halo=df.halo))
    plist, out["prune"] = t(lambda: prune_pair_list(built, grid.clustered_positions_device, s.box, r_inner=0.0))
    df.grid, df.plist = grid, plist
    df.f = torch.empty((lay.n_local, 3), dtype=torch.float64, device=dev)
    _, out["first_force(layout)"] = t(lambda: df.forces(energy=False))
    return lay, out


for rep in range(4):
    glob, t_ag = t(lambda: dd.allgather_home(lay.home, df.local_pos[:lay.n_home], s.n))
    lay, ph = rebuild_phases(glob)
    if rank == 0:
        print(f"N={world} rep {rep} phases (ms): allgather {t_ag:.3f} " + " ".join(f"{k} {v:.3f}" for k, v in ph.items()))
    glob, t_ag = t(lambda: dd.allgather_home(lay.home, df.local_pos[:lay.n_home], s.n))
    _, t_as = t(lambda: dd.assign(glob))
    lay, t_rb = t(lambda: df.rebuild(glob))
    _, t_f1 = t(lambda: df.forces(energy=True))
    _, t_f2 = t(lambda: df.forces(energy=False))
    if rank == 0:
        print(f"N={world} rep {rep}: allgather {t_ag:.3f} ms | assign {t_as:.3f} | rebuild(incl assign) {t_rb:.3f} | "
              f"force#1 {t_f1:.3f} | force {t_f2:.3f} | home {lay.n_home} halo {lay.n_local - lay.n_home}")

# host enqueue cost vs device time of force-only steps (host-bound if close)
torch.cuda.synchronize()
dist.barrier()
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ev0.record()
h0 = time.perf_counter()
for _ in range(50):
    df.forces(energy=False)
h1 = time.perf_counter()
ev1.record()
torch.cuda.synchronize()
if rank == 0:
    print(f"N={world} force steps: host enqueue {1e6 * (h1 - h0) / 50:.1f} us/step, "
          f"device {1e3 * ev0.elapsed_time(ev1) / 50:.1f} us/step")
dist.destroy_process_group()
