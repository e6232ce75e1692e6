"""Two-step (build_pair_list + prune_pair_list) vs fused
(build_pruned_pair_list) list construction: device time of each, lists
compared.   python tools/list_step_ab.py [atoms]"""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1506_00716_b200 as nbx  # noqa: E402
from paper_1506_00716_b200.systems import spc_water, tuned_occupancy  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 96000
s, table = spc_water(n)
occ = tuned_occupancy(n, float(s.box.lengths[0]), 4)
pos = torch.from_numpy(np.array(s.positions)).cuda()


def timed(fn, reps=5):
    out = None
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return out, 1e3 * min(ts)


grid, tg = timed(lambda: nbx.build_cluster_grid(s, 4, occ, positions=pos))
two, t2 = timed(lambda: nbx.prune_pair_list(nbx.build_pair_list(grid, s.box, 1.1), grid.clustered_positions_device,
                                            s.box))
fused, tf = timed(lambda: nbx.build_pruned_pair_list(grid, s.box, 1.1))
same = np.array_equal(two.offsets, fused.offsets) and np.array_equal(two.j_idx, fused.j_idx) and \
    np.array_equal(two.mask_bits, fused.mask_bits)
print(f"atoms {n}: grid {tg:.3f} ms, build+prune {t2:.3f} ms, fused {tf:.3f} ms, identical {same}")
