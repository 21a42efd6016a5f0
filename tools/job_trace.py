import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_2309_14311_b200 import nasch
L, N = 10**9, 2 * 10**8
x, v = nasch.fill_uniform_state(L, N, 0, 3)
def pinned(a=None, n=N):
    t = torch.zeros(n, dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
    if a is not None: t[:] = a
    return t
xin, vin = pinned(x), pinned(v)
outx, outv = pinned(), pinned()
for rep in range(4):
    e = nasch.Engine(nasch.SimParams(length=L, ncars=N, vmax=5, p=0.13, steps=100, seed=3))
    e.set_checksum(False)
    t0 = time.perf_counter()
    e.job32(xin, vin, 20, out_x=outx, out_v=outv)
    print(f"job32 {1e3*(time.perf_counter()-t0):.2f} ms", flush=True)
    e.close()
# raw PCIe: H2D 0.8 GB and D2H 0.8 GB alone and together
d = torch.empty(N, dtype=torch.int32, device='cuda'); d2 = torch.empty(N, dtype=torch.int32, device='cuda')
tx = torch.from_numpy(xin.view(np.int32)); to = torch.from_numpy(outx.view(np.int32))
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for name, fn in [("h2d", lambda: d.copy_(tx, non_blocking=True)), ("d2h", lambda: to.copy_(d2, non_blocking=True))]:
    torch.cuda.synchronize(); t0 = time.perf_counter(); fn(); torch.cuda.synchronize()
    dt = time.perf_counter() - t0; print(name, f"{1e3*dt:.2f} ms {0.8/dt:.1f} GB/s")
torch.cuda.synchronize(); t0 = time.perf_counter()
with torch.cuda.stream(s1): d.copy_(tx, non_blocking=True)
with torch.cuda.stream(s2): to.copy_(d2, non_blocking=True)
torch.cuda.synchronize(); dt = time.perf_counter() - t0; print("both", f"{1e3*dt:.2f} ms")
print("cores", os.cpu_count())
