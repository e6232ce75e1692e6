"""Force pass at cluster size m = 4 vs 8 on the bench box (96k SPC, Ewald):
device time per pass (CUDA events, 20 passes), admitted / within pairs,
useful pairs/s.   python tools/m_compare.py [atoms]"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1506_00716_b200 as nbx  # noqa: E402
from paper_1506_00716_b200.systems import spc_water, tuned_occupancy  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 96000
s, table = spc_water(n)
params = nbx.NonbondedParams(r_cut=1.0, r_list=1.1, lj_table=table, shift_potential=True, elec="ewald",
                             ewald_beta=nbx.ewald_beta(1.0))
pos = torch.from_numpy(np.array(s.positions)).cuda()
q = torch.from_numpy(np.array(s.charges)).cuda()
t = torch.from_numpy(np.array(s.lj_type)).cuda()
f = torch.empty_like(pos)
for m in (4, 8):
    for occ_name, occ in (("tuned", tuned_occupancy(n, float(s.box.lengths[0]), m)), ("default", None)):
        g, p = nbx.list_step(s, m, occ, s.box, 1.1, positions=pos)
        st = nbx.interaction_stats(p, g, g.clustered_positions_device, s.box, 1.0)
        for _ in range(3):
            nbx.compute_nonbonded_device(p, g, pos, q, t, params, s.box, energy=False, out=f)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            nbx.compute_nonbonded_device(p, g, pos, q, t, params, s.box, energy=False, out=f)
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / 20 * 1e3
        print(f"m={m} {occ_name:7s} pass {us:6.1f} us  admitted {st.n_admitted / 1e6:5.1f} M  within "
              f"{st.n_within_cutoff / 1e6:5.1f} M  useful {st.n_within_cutoff / us / 1e3:6.1f} G/s  "
              f"admitted {st.n_admitted / us / 1e3:6.1f} G/s")
