"""Device time of the list step (pairlist.list_step: grid + search + prune +
force layout) and of its search kernels, CUDA events, mean of 20 after 5
warm-ups.  A/B library builds with NBX_LIB=...
    python tools/list_step_time.py [atoms ...]"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1506_00716_b200 as nbx  # noqa: E402
from paper_1506_00716_b200 import _lib  # noqa: E402
from paper_1506_00716_b200.systems import spc_water, tuned_occupancy  # noqa: E402

for n in [int(a) for a in sys.argv[1:]] or [96000]:
    s, _ = spc_water(n)
    occ = tuned_occupancy(n, float(s.box.lengths[0]), 4)
    pos = torch.from_numpy(np.array(s.positions)).cuda()
    for _ in range(5):
        g, p = nbx.list_step(s, 4, occ, s.box, 1.1, positions=pos)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    lib = _lib.load()
    lib.nbx_timing_query(None, None)
    e0.record()
    for _ in range(20):
        g, p = nbx.list_step(s, 4, occ, s.box, 1.1, positions=pos)
    e1.record()
    torch.cuda.synchronize()
    print(f"{n} atoms: list step {e0.elapsed_time(e1) / 20 * 1e3:.1f} us (wall, incl. host syncs), "
          f"{p.n_entries} entries")
