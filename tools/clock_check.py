"""NVML clock / throttle sampling check of bench.Clocks on the GPU box."""
import sys, time
sys.path.insert(0, "/root/repo")
import faulthandler; faulthandler.enable()
import torch
torch.cuda.set_device(0)
import bench
c = bench.Clocks(0)
x = torch.randn(4096, 4096, device="cuda")
for _ in range(50): x = x @ x; x = x / x.norm()
torch.cuda.synchronize()
print(c.stop())
