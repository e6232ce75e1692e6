"""Kernel timeline of rigid-water run_md steps (96k SPC, the bench's MD):
device time per kernel, GPU idle, CUDA runtime calls (torch.profiler).
    python tools/md_trace.py [--atoms 96000] [--steps 40]"""
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
ap.add_argument("--steps", type=int, default=200)
a = ap.parse_args()
system, table = spc_water(a.atoms, seed=2024, temperature=300.0)
occ = tuned_occupancy(a.atoms, float(system.box.lengths[0]), 4)
params = nbx.NonbondedParams(r_cut=1.0, r_list=1.1, lj_table=table, shift_potential=True, elec="ewald",
                             ewald_beta=nbx.ewald_beta(1.0))
water, layout = nbx.RigidWater(), nbx.KernelLayout(4, 4)
res = nbx.run_md(system, params, layout, 0.002, 100, report_interval=10, target_occupancy=occ, constraints=water)
system = res.state.system
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CPU,
                                        torch.profiler.ProfilerActivity.CUDA]) as prof:
    res = nbx.run_md(system, params, layout, 0.002, a.steps, report_interval=10, target_occupancy=occ,
                     constraints=water)
    torch.cuda.synchronize()
print(f"{a.steps} steps, {res.state.n_rebuilds} rebuilds ({res.state.n_drift_rebuilds} by the drift guard)")
out = Path("gpurun_out")
out.mkdir(exist_ok=True)
prof.export_chrome_trace(str(out / "md_trace.json"))
ev = json.load(open(out / "md_trace.json"))["traceEvents"]
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
# steady state: from the first integrator kernel (after run_md's setup)
k0 = next(i for i, k in enumerate(kern) if "k_vv" in k[2])
kern = kern[k0:]
span = kern[-1][1] - kern[0][0]
busy, end, gaps = 0.0, kern[0][0], []
for t0, t1, name in kern:
    if t0 > end:
        gaps.append((t0 - end, name))
    busy += max(0.0, t1 - max(t0, end))
    end = max(end, t1)
S = a.steps
print(f"span {span / S:.1f} us/step, kernels busy {busy / S:.1f}, idle {(span - busy) / S:.1f} us/step")
tot = defaultdict(lambda: [0, 0.0])
for t0, t1, name in kern:
    tot[name.split("(")[0][:70]][0] += 1
    tot[name.split("(")[0][:70]][1] += t1 - t0
for k, (c, d) in sorted(tot.items(), key=lambda x: -x[1][1])[:30]:
    print(f"   {c:5d} {d / S:8.1f} us/step  {k}")
big = sorted(gaps, reverse=True)[:12]
print("largest gaps:", ", ".join(f"{g:.0f}us<{n.split('(')[0][:28]}" for g, n in big))
gsum = defaultdict(float)
for g, n in gaps:
    gsum[n.split("(")[0][:40]] += g
print("idle before (sum/step):", ", ".join(f"{n} {v / S:.1f}" for n, v in sorted(gsum.items(), key=lambda x: -x[1])[:12]))
print("runtime:", ", ".join(f"{k} {c}x {d / S:.0f}us/step" for k, (c, d) in sorted(rt.items(), key=lambda x: -x[1][1])[:10]))
