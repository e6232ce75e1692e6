"""Where the host time of a list rebuild goes (Python wrapper vs C entry)."""
import ctypes
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
acc = {}


def wrap(name):
    fn = getattr(lib, name)

    def w(*a):
        t0 = time.perf_counter()
        r = fn(*a)
        acc[name] = acc.get(name, 0.0) + time.perf_counter() - t0
        return r
    return w


class L:  # proxy recording the C entry time
    def __getattr__(self, k):
        return wrap(k)


_lib.load = lambda: L()
tot = {}
keep = []
for rep in range(23):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    g = nbx.build_cluster_grid(s, 4, occ, positions=pos)
    t1 = time.perf_counter()
    b = nbx.build_pair_list(g, s.box, 1.1)
    t2 = time.perf_counter()
    p = nbx.prune_pair_list(b, g.clustered_positions_device, s.box)
    t3 = time.perf_counter()
    del b
    t4 = time.perf_counter()
    keep = [g, p]   # the previous generation is released here
    t5 = time.perf_counter()
    if rep >= 3:
        for k, v in (("grid", t1 - t0), ("build", t2 - t1), ("prune", t3 - t2), ("del built", t4 - t3),
                     ("release previous", t5 - t4)):
            tot[k] = tot.get(k, 0.0) + v
for k, v in tot.items():
    print(f"{k:18s} {1e6 * v / 20:8.1f} us")
for k, v in sorted(acc.items(), key=lambda x: -x[1]):
    print(f"  C {k:28s} {1e6 * v / 23:8.1f} us")
