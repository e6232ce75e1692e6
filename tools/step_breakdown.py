"""Per-phase timing of one rebuild + force passes (CUDA events and wall clock).

    python tools/step_breakdown.py [--atoms 96000] [--elec ewald]
"""

import argparse
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1506_00716_b200 as nbx  # noqa: E402
from paper_1506_00716_b200.systems import spc_water, tuned_occupancy  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--atoms", type=int, default=96000)
    ap.add_argument("--elec", default="ewald")
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    s, table = spc_water(a.atoms)
    L = float(s.box.lengths[0])
    occ = tuned_occupancy(a.atoms, L, 4)
    if a.elec == "ewald":
        params = nbx.NonbondedParams(r_cut=1.0, r_list=1.1, lj_table=table, shift_potential=True, elec="ewald",
                                     ewald_beta=nbx.ewald_beta(1.0))
    else:
        params = nbx.NonbondedParams(r_cut=1.0, r_list=1.1, lj_table=table, shift_potential=True)
    dev = torch.device("cuda", 0)
    pos = torch.from_numpy(np.array(s.positions)).to(dev)
    q = torch.from_numpy(np.array(s.charges)).to(dev)
    t = torch.from_numpy(np.array(s.lj_type)).to(dev)
    out = torch.empty((s.n, 3), dtype=torch.float64, device=dev)

    def timed(fn):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        w0 = time.perf_counter()
        e0.record()
        r = fn()
        e1.record()
        torch.cuda.synchronize()
        return r, e0.elapsed_time(e1), 1e3 * (time.perf_counter() - w0)

    for rep in range(a.reps):
        grid, g_ms, g_w = timed(lambda: nbx.build_cluster_grid(s, 4, occ, positions=pos))
        built, b_ms, b_w = timed(lambda: nbx.build_pair_list(grid, s.box, 1.1))
        pl, p_ms, p_w = timed(lambda: nbx.prune_pair_list(built, grid.clustered_positions_device, s.box))
        pf, bp_ms, bp_w = timed(lambda: nbx.build_pruned_pair_list(grid, s.box, 1.1))
        _, f1_ms, f1_w = timed(lambda: nbx.compute_nonbonded_device(pl, grid, pos, q, t, params, s.box, out=out))
        _, f2_ms, f2_w = timed(lambda: nbx.compute_nonbonded_device(pl, grid, pos, q, t, params, s.box, out=out,
                                                                     energy=False))
        print(f"rep {rep}: grid {g_ms:.3f} ms (wall {g_w:.3f}) | build {b_ms:.3f} ({b_w:.3f}) | prune {p_ms:.3f} "
              f"({p_w:.3f}) | build_pruned {bp_ms:.3f} | force#1 {f1_ms:.3f} ({f1_w:.3f}) | force {f2_ms:.3f} ({f2_w:.3f})")
    print(f"rows built {built.n_pairs} pruned {pl.n_pairs} groups {pl.n_groups} entries {pl.n_entries}")


if __name__ == "__main__":
    main()
