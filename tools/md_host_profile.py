"""cProfile of 400 rigid-water run_md steps at 96k (host time per call of the MD loop)."""
import sys, cProfile, pstats; sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_1506_00716_b200 as nbx
from paper_1506_00716_b200.systems import spc_water, tuned_occupancy
system, table = spc_water(96000, seed=2024, temperature=300.0)
occ = tuned_occupancy(96000, float(system.box.lengths[0]), 4)
params = nbx.NonbondedParams(r_cut=1.0, r_list=1.1, lj_table=table, shift_potential=True, elec="ewald", ewald_beta=nbx.ewald_beta(1.0))
water, layout = nbx.RigidWater(), nbx.KernelLayout(4, 4)
res = nbx.run_md(system, params, layout, 0.002, 100, report_interval=10, target_occupancy=occ, constraints=water)
system = res.state.system
pr = cProfile.Profile(); pr.enable()
res = nbx.run_md(system, params, layout, 0.002, 400, report_interval=10, target_occupancy=occ, constraints=water)
torch.cuda.synchronize()
pr.disable()
print("rebuilds", res.state.n_rebuilds)
pstats.Stats(pr).sort_stats("tottime").print_stats(30)
