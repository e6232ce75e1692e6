"""Timeline of rigid-water MD steps around list rebuilds (torch.profiler /
CUPTI): every CUDA runtime call the library makes (syncs, copies, launches)
and every kernel, so GPU idle gaps can be attributed.

    python tools/rebuild_trace.py [--atoms 96000] [--steps 12]
    -> gpurun_out/rebuild_trace.json (chrome trace) + a summary on stdout"""
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
ap.add_argument("--steps", type=int, default=12)
a = ap.parse_args()
s, table = spc_water(a.atoms, seed=2024, temperature=300.0)
occ = tuned_occupancy(a.atoms, float(s.box.lengths[0]), 4)
params = nbx.NonbondedParams(r_cut=1.0, r_list=1.1, lj_table=table, shift_potential=True, elec="ewald",
                             ewald_beta=nbx.ewald_beta(1.0))
layout = nbx.KernelLayout(4, 4)
water = nbx.RigidWater()
import dataclasses  # noqa: E402

for _ in range(5):  # relax the lattice and bring it to 300 K (as bench.py)
    r = nbx.run_md(s, params, layout, 0.002, 20, report_interval=20, target_occupancy=occ, constraints=water)
    s = dataclasses.replace(r.state.system, velocities=r.state.system.velocities * np.sqrt(
        300.0 / max(float(r.temperature[-1]), 1.0)))
torch.cuda.synchronize()
acts = [torch.profiler.ProfilerActivity.CPU, torch.profiler.ProfilerActivity.CUDA]
with torch.profiler.profile(activities=acts) as prof:
    res = nbx.run_md(s, params, layout, 0.002, a.steps, report_interval=10, target_occupancy=occ, constraints=water)
    torch.cuda.synchronize()
out = Path("gpurun_out")
out.mkdir(exist_ok=True)
prof.export_chrome_trace(str(out / "rebuild_trace.json"))
ev = json.load(open(out / "rebuild_trace.json"))["traceEvents"]
rt = defaultdict(lambda: [0, 0.0])
kern = []
for e in ev:
    if e.get("ph") != "X":
        continue
    cat = e.get("cat", "")
    if cat == "cuda_runtime" or cat == "cuda_driver":
        rt[e["name"]][0] += 1
        rt[e["name"]][1] += e.get("dur", 0)
    elif cat == "kernel" or cat == "gpu_memcpy" or cat == "gpu_memset":
        kern.append((e["ts"], e["ts"] + e.get("dur", 0), e["name"]))
kern.sort()
# steady state only: from the first integrator kernel to the last RATTLE
t_first = min(t0 for t0, _, n in kern if "k_vv" in n)
t_last = max(t1 for _, t1, n in kern if "k_rattle_v" in n)
kern = [k for k in kern if t_first <= k[0] <= t_last]
busy = 0.0
gaps = []
end = kern[0][0] if kern else 0
for t0, t1, name in kern:
    if t0 > end:
        gaps.append((t0 - end, name))
    busy += max(0.0, t1 - max(t0, end))
    end = max(end, t1)
span = kern[-1][1] - kern[0][0] if kern else 0
print(f"steps {a.steps}: rebuilds {res.state.n_rebuilds}, device span {span:.0f} us, busy {busy:.0f} us "
      f"({100 * busy / max(span, 1):.0f} %), idle {span - busy:.0f} us")
print("largest GPU idle gaps (us, next activity):")
for g, name in sorted(gaps, reverse=True)[:15]:
    print(f"  {g:8.1f}  {name[:90]}")
print("CUDA runtime calls (count, total us):")
for k, (c, d) in sorted(rt.items(), key=lambda x: -x[1][1])[:15]:
    print(f"  {c:6d} {d:10.0f}  {k}")

tot = defaultdict(lambda: [0, 0.0])
for t0, t1, name in kern:
    key = name.split("(")[0][:80]
    tot[key][0] += 1
    tot[key][1] += t1 - t0
print("device time by kernel in the window (count, total us):")
for k, (c, d) in sorted(tot.items(), key=lambda x: -x[1][1])[:30]:
    print(f"  {c:5d} {d:9.1f}  {k}")
