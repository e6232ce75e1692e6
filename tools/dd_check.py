"""Multi-GPU parity: slab-decomposed forces/energies vs one GPU (torchrun, NCCL).

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/dd_check.py [--atoms 96000]
"""
import argparse
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

ap = argparse.ArgumentParser()
ap.add_argument("--atoms", type=int, default=96000)
ap.add_argument("--torch-p2p", action="store_true")
ap.add_argument("--p2p", action="store_true", help="NVLink peer-store exchanges (overlapped with the force pass)")
a = ap.parse_args()
rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
import datetime
dist.init_process_group("nccl", device_id=torch.device("cuda", local), timeout=datetime.timedelta(seconds=90))
s, table = spc_water(a.atoms)
L = s.box.lengths
occ = tuned_occupancy(a.atoms, float(L[0]), 4)
params = nbx.NonbondedParams(r_cut=1.0, r_list=1.1, lj_table=table, shift_potential=True, elec="ewald",
                             ewald_beta=nbx.ewald_beta(1.0))
dev = torch.device("cuda", local)
pos = torch.from_numpy(np.array(s.positions)).to(dev)
dd = SlabDecomposition(L, world, rank, r_comm=1.1)
if '--torch-p2p' not in sys.argv:
    dd.enable_native()
    if a.p2p:
        print(f"rank {rank}: p2p {dd.enable_p2p(s.n)}")
df_overlap = a.p2p
df = DomainForces(dd, s, params, 4, occ)
lay = df.rebuild(pos)
df.overlap = a.p2p  # the overlapped nbx_dd_force path
home_f, e = df.forces(energy=True)
glob = dd.allgather_home(lay.home, home_f, s.n)
st = nbx.interaction_stats(df.plist, df.grid, df.grid.clustered_positions_device, s.box, 1.0)
tot = torch.tensor([st.n_within_cutoff], dtype=torch.int64, device=dev)
dist.all_reduce(tot)
if rank == 0:
    grid = nbx.build_cluster_grid(s, 4, occ)
    pl = nbx.prune_pair_list(nbx.build_pair_list(grid, s.box, 1.1), grid.clustered_positions, s.box)
    ref = nbx.compute_nonbonded_original(pl, grid, s.positions, s.charges, s.lj_type, params, s.box,
                                         nbx.KernelLayout(4, 4))
    f = glob.cpu().numpy()
    rr = np.sqrt(((f - ref.forces) ** 2).sum() / (ref.forces ** 2).sum())
    e = e.cpu().numpy()
    n1 = nbx.interaction_stats(pl, grid, grid.clustered_positions, s.box, 1.0).n_within_cutoff
    print(f"world {world}: force rel-RMS vs 1 GPU {rr:.2e}; e_lj {e[0]:.6f} vs {ref.e_lj:.6f}; "
          f"e_c {e[1]:.6f} vs {ref.e_coulomb:.6f}; pairs within r_c {int(tot.item())} vs {n1}")
    ok = rr < 1e-5 and abs(e[0] - ref.e_lj) < 1e-6 * abs(ref.e_lj) and abs(e[1] - ref.e_coulomb) < 1e-6 * abs(ref.e_coulomb) \
        and int(tot.item()) == n1
    print("DD PARITY", "OK" if ok else "FAIL")
dist.destroy_process_group()
