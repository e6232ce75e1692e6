"""Host time of each piece of a 96k list rebuild (median over reps, µs):
the C entry points vs the Python around them.   python tools/host_gaps.py"""
import statistics
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1506_00716_b200 as nbx  # noqa: E402
from paper_1506_00716_b200 import _lib  # noqa: E402
from paper_1506_00716_b200.systems import spc_water, tuned_occupancy  # noqa: E402

s, table = spc_water(96000)
occ = tuned_occupancy(96000, float(s.box.lengths[0]), 4)
pos = torch.from_numpy(np.array(s.positions)).to("cuda")
lib = _lib.load()
rec = {}


class Wrap:
    def __getattr__(self, k):
        fn = getattr(lib, k)

        def w(*a):
            t0 = time.perf_counter()
            r = fn(*a)
            rec.setdefault("C " + k, []).append(1e6 * (time.perf_counter() - t0))
            return r
        return w


_lib.load = lambda: Wrap()
keep = None
for rep in range(25):
    torch.cuda.synchronize()
    t = [time.perf_counter()]
    g = nbx.build_cluster_grid(s, 4, occ, positions=pos)
    t.append(time.perf_counter())
    b = nbx.build_pair_list(g, s.box, 1.1)
    t.append(time.perf_counter())
    p = nbx.prune_pair_list(b, g.clustered_positions_device, s.box, r_inner=1.02)
    t.append(time.perf_counter())
    del b
    t.append(time.perf_counter())
    keep = (g, p)
    t.append(time.perf_counter())
    torch.cuda.synchronize()
    t.append(time.perf_counter())
    for name, a, z in (("grid", 0, 1), ("build", 1, 2), ("prune", 2, 3), ("del built", 3, 4), ("release prev", 4, 5),
                       ("drain", 5, 6)):
        rec.setdefault(name, []).append(1e6 * (t[z] - t[a]))
for k, v in rec.items():
    v = v[5:] if len(v) > 10 else v
    print(f"{k:34s} median {statistics.median(v):9.1f} us  max {max(v):9.1f}  n {len(v)}")
