"""Kernel-level timeline of the list step (grid, search, prune, first force
pass with the force-layout set-up) on the bench box: device time per kernel,
GPU idle gaps, CUDA runtime calls (torch.profiler / CUPTI).
    python tools/list_step_trace.py [--atoms 96000] [--reps 3]"""
import argparse
import json
import sys
from collections import defaultdict
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1506_00716_b200 as nbx  # noqa: E402
from paper_1506_00716_b200.systems import spc_water, tuned_occupancy  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--atoms", type=int, default=96000)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--md", type=int, default=0, help="take positions after this many rigid-water run_md steps")
a = ap.parse_args()
s, table = spc_water(a.atoms)
occ = tuned_occupancy(a.atoms, float(s.box.lengths[0]), 4)
params = nbx.NonbondedParams(r_cut=1.0, r_list=1.1, lj_table=table, shift_potential=True, elec="ewald",
                             ewald_beta=nbx.ewald_beta(1.0))
if a.md:
    s, _ = spc_water(a.atoms, seed=2024, temperature=300.0)
    s = nbx.run_md(s, params, nbx.KernelLayout(4, 4), 0.002, a.md, report_interval=a.md, target_occupancy=occ,
                   constraints=nbx.RigidWater()).state.system
dev = torch.device("cuda", 0)
pos = torch.from_numpy(np.array(s.positions)).to(dev)
q = torch.from_numpy(np.array(s.charges)).to(dev)
t = torch.from_numpy(np.array(s.lj_type)).to(dev)
f = torch.empty_like(pos)


def list_step():
    grid = nbx.build_cluster_grid(s, 4, occ, positions=pos)
    pl = nbx.prune_pair_list(nbx.build_pair_list(grid, s.box, 1.1), grid.clustered_positions_device, s.box)
    nbx.compute_nonbonded_device(pl, grid, pos, q, t, params, s.box, energy=False, out=f)
    return grid, pl


for _ in range(3):
    list_step()
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CPU,
                                        torch.profiler.ProfilerActivity.CUDA]) as prof:
    for _ in range(a.reps):
        keep = list_step()
        torch.cuda.synchronize()
out = Path("gpurun_out")
out.mkdir(exist_ok=True)
prof.export_chrome_trace(str(out / "list_step_trace.json"))
ev = json.load(open(out / "list_step_trace.json"))["traceEvents"]
kern, rt = [], defaultdict(lambda: [0, 0.0])
for e in ev:
    if e.get("ph") != "X":
        continue
    cat = e.get("cat", "")
    if cat in ("kernel", "gpu_memcpy", "gpu_memset"):
        kern.append((e["ts"], e["ts"] + e.get("dur", 0), e["name"]))
    elif cat in ("cuda_runtime", "cuda_driver"):
        rt[e["name"]][0] += 1
        rt[e["name"]][1] += e.get("dur", 0)
kern.sort()
# split into reps at the k_bin kernels (first kernel of each grid build)
starts = [i for i, k in enumerate(kern) if "k_bin" in k[2]]
starts.append(len(kern))
for r in range(len(starts) - 1):
    ks = kern[starts[r]:starts[r + 1]]
    span = ks[-1][1] - ks[0][0]
    busy, end, gaps = 0.0, ks[0][0], []
    for t0, t1, name in ks:
        if t0 > end:
            gaps.append((t0 - end, name))
        busy += max(0.0, t1 - max(t0, end))
        end = max(end, t1)
    print(f"list step {r}: span {span:.0f} us, kernels busy {busy:.0f} us, idle {span - busy:.0f} us, "
          f"{len(ks)} device activities")
    if r == len(starts) - 2:
        tot = defaultdict(lambda: [0, 0.0])
        for t0, t1, name in ks:
            tot[name.split("(")[0][:70]][0] += 1
            tot[name.split("(")[0][:70]][1] += t1 - t0
        for k, (c, d) in sorted(tot.items(), key=lambda x: -x[1][1])[:24]:
            print(f"   {c:3d} {d:8.1f} us  {k}")
        print("  largest gaps:", ", ".join(f"{g:.0f}us<{n.split('(')[0][:30]}" for g, n in sorted(gaps, reverse=True)[:8]))
print("runtime:", ", ".join(f"{k} {c}x {d:.0f}us" for k, (c, d) in sorted(rt.items(), key=lambda x: -x[1][1])[:8]))
