"""Kernel timeline of the bench's force-only steps (96k SPC, moving
trajectory, current list; drift guard + force pass as bench.py run_ours):
device time per kernel and the GPU idle between them.
    python tools/force_step_trace.py [steps]"""
import json
import sys
from collections import defaultdict
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402
import paper_1506_00716_b200 as nbx  # noqa: E402
from paper_1506_00716_b200.engine import max_displacement_device  # noqa: E402
from paper_1506_00716_b200.systems import spc_water, tuned_occupancy  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 30
s, table = spc_water(96000)
occ = tuned_occupancy(96000, float(s.box.lengths[0]), 4)
params = nbx.NonbondedParams(r_cut=1.0, r_list=1.1, lj_table=table, shift_potential=True, elec="ewald",
                             ewald_beta=nbx.ewald_beta(1.0))
traj = bench.Trajectory(s)
dev = torch.device("cuda", 0)
traj.to_device(dev, range(0, K + 10))
q = torch.from_numpy(np.array(s.charges)).to(dev)
t = torch.from_numpy(np.array(s.lj_type)).to(dev)
f = torch.empty((s.n, 3), dtype=torch.float64, device=dev)
e = torch.zeros(2, dtype=torch.float64, device=dev)
bad = torch.empty(2, dtype=torch.int64, device=dev)
ref = traj.device(0).clone()
grid, plist = nbx.list_step(s, 4, occ, s.box, 1.1, positions=ref)
d_pin = torch.zeros(1, dtype=torch.float64).pin_memory()


def step(k):
    pos = traj.device(k)
    d_pin.copy_(max_displacement_device(ref, pos, s.box), non_blocking=True)
    nbx.compute_nonbonded_device(plist, grid, pos, q, t, params, s.box, energy=False, out=f, e_out=e, bad=bad)


for k in range(1, 6):
    step(k)
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    for k in range(6, 6 + K):
        step(k)
    torch.cuda.synchronize()
Path("gpurun_out").mkdir(exist_ok=True)
prof.export_chrome_trace("gpurun_out/force_step_trace.json")
ev = json.load(open("gpurun_out/force_step_trace.json"))["traceEvents"]
kern = sorted((x["ts"], x["ts"] + x.get("dur", 0), x["name"]) for x in ev
              if x.get("ph") == "X" and x.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset"))
span = kern[-1][1] - kern[0][0]
busy, end = 0.0, kern[0][0]
gaps = defaultdict(float)
for t0, t1, name in kern:
    if t0 > end:
        gaps[name.split("(")[0][:50]] += t0 - end
    busy += max(0.0, t1 - max(t0, end))
    end = max(end, t1)
print(f"{K} force steps: span {span / K:.1f} us/step, busy {busy / K:.1f}, idle {(span - busy) / K:.1f} us/step, "
      f"{len(kern) / K:.1f} device activities per step")
tot = defaultdict(lambda: [0, 0.0])
for t0, t1, name in kern:
    tot[name.split("(")[0][:60]][0] += 1
    tot[name.split("(")[0][:60]][1] += t1 - t0
for k_, (c, d) in sorted(tot.items(), key=lambda x: -x[1][1]):
    print(f"   {c // K:3d}x {d / K:8.1f} us/step  {k_}")
print("idle before (us/step):", ", ".join(f"{n} {v / K:.1f}" for n, v in sorted(gaps.items(), key=lambda x: -x[1])))
