"""Host (CUDA runtime API) and device events of one list rebuild, one timeline:
where the GPU waits for the host.   python tools/timeline_host.py"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1506_00716_b200 as nbx  # noqa: E402
from paper_1506_00716_b200.systems import spc_water, tuned_occupancy  # noqa: E402

s, table = spc_water(96000)
occ = tuned_occupancy(96000, float(s.box.lengths[0]), 4)
dev = torch.device("cuda", 0)
pos = torch.from_numpy(np.array(s.positions)).to(dev)


def rebuild():
    grid = nbx.build_cluster_grid(s, 4, occ, positions=pos)
    return grid, nbx.prune_pair_list(nbx.build_pair_list(grid, s.box, 1.1), grid.clustered_positions_device, s.box)


for _ in range(3):
    rebuild()
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    rebuild()
    torch.cuda.synchronize()
ev = sorted(prof.events(), key=lambda x: x.time_range.start)
t0 = ev[0].time_range.start
for x in ev:
    side = "GPU" if x.device_type == torch.autograd.DeviceType.CUDA else "cpu"
    print(f"{x.time_range.start - t0:9.1f} {x.time_range.end - x.time_range.start:8.1f} {side} {x.name[:70]}")
