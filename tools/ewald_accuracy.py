"""Force / energy error of the GPU path vs the FP64 oracle (24k SPC, 3 physics)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1506_00716_b200 as nbx  # noqa: E402
from oracle import forces as of  # noqa: E402
from oracle import native, search  # noqa: E402
from paper_1506_00716_b200.systems import spc_water, tuned_occupancy  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 24000
s, table = spc_water(n)
L = s.box.lengths
occ = tuned_occupancy(n, float(L[0]), 4)
grid = nbx.build_cluster_grid(s, 4, occ)
pl = nbx.prune_pair_list(nbx.build_pair_list(grid, s.box, 1.1), grid.clustered_positions, s.box)
og = search.build_grid(s.positions, L, 4, occ)
ol = dict(m=4, offsets=pl.offsets, j_idx=pl.j_idx, masks=pl.masks, r_list=1.1)
beta = nbx.ewald_beta(1.0)
for name, kw in (("cutoff", {}), ("rf_inf", dict(elec="reaction_field", epsilon_rf=0.0)),
                 ("ewald", dict(elec="ewald", ewald_beta=beta))):
    params = nbx.NonbondedParams(r_cut=1.0, r_list=1.1, lj_table=table, shift_potential=True, **kw)
    phys = of.Physics(r_cut=1.0, lj_table=table, shift_potential=True, **kw)
    res = nbx.compute_nonbonded_original(pl, grid, s.positions, s.charges, s.lj_type, params, s.box,
                                         nbx.KernelLayout(4, 4))
    fc, elj, ec = native.list_forces(ol, og, s.positions, s.charges, s.lj_type, L, phys)
    fr = search.scatter_to_original(og, fc)
    rr = np.sqrt(((res.forces - fr) ** 2).sum() / (fr ** 2).sum())
    print(f"{name:8s} force rel-RMS {rr:.2e}  e_lj rel {abs(res.e_lj - elj) / abs(elj):.2e}  "
          f"e_c rel {abs(res.e_coulomb - ec) / abs(ec):.2e}")
