"""Host copies of a 96k x 3 FP64 array: numpy into / out of pinned memory with 1-8 threads, pinned H2D / D2H,
tensor.cpu() (the drop-in path's transfer budget)."""
import time, numpy as np, torch
from concurrent.futures import ThreadPoolExecutor
n = 96000
src = np.random.rand(n, 3)
pin = torch.empty(n * 3, dtype=torch.float64).pin_memory()
pv = pin.numpy()
pool = ThreadPoolExecutor(8)
def tm(f, k=50):
    f(); t0 = time.perf_counter()
    for _ in range(k): f()
    return (time.perf_counter() - t0) / k * 1e6
def par_copy(dst, s, parts):
    d = dst.reshape(-1); s = s.reshape(-1); m = d.size
    b = [m * i // parts for i in range(parts + 1)]
    list(pool.map(lambda i: np.copyto(d[b[i]:b[i+1]], s[b[i]:b[i+1]]), range(parts)))
print("copyto into pinned 1 thread us", tm(lambda: np.copyto(pv, src.reshape(-1))))
for p in (2, 4, 8):
    print(f"copyto into pinned {p} threads us", tm(lambda: par_copy(pv, src, p)))
print("fresh empty + copy from pinned 1 thread", tm(lambda: pv.copy()))
def fresh_par(p):
    out = np.empty(n * 3); par_copy(out, pv, p); return out
for p in (2, 4, 8):
    print(f"fresh empty + copy {p} threads", tm(lambda: fresh_par(p)))
d = torch.empty(n * 3, dtype=torch.float64, device="cuda")
def h2d():
    d.copy_(pin, non_blocking=True); torch.cuda.current_stream().synchronize()
print("H2D 2.3MB pinned", tm(h2d))
def d2h():
    pin.copy_(d, non_blocking=True); torch.cuda.current_stream().synchronize()
print("D2H 2.3MB pinned", tm(d2h))
print("tensor.cpu()", tm(lambda: d.cpu()))
