"""Host-transfer legs of the end-to-end path on BASELINE config 3 (one GPU):
set_state32 from pinned int32 arrays, the velocity series, state32 into
pinned int32 arrays, each timed alone (wall clock, 3 repeats).
    python tools/e2e_probe.py"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2309_14311_b200 import nasch  # noqa: E402

L, N = 10**9, 2 * 10**8
x, v = nasch.fill_uniform_state(L, N, 0, 3)


def pinned(a=None, n=N):
    t = torch.zeros(n, dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
    if a is not None:
        t[:] = a
    return t


xin, vin = pinned(x), pinned(v)
outx, outv = pinned(), pinned()
e = nasch.Engine(nasch.SimParams(length=L, ncars=N, vmax=5, p=0.13, steps=100, seed=3))
e.set_checksum(False)
for rep in range(3):
    t0 = time.perf_counter()
    e.set_state(xin, vin)
    t1 = time.perf_counter()
    e.advance(20)
    t2 = time.perf_counter()
    s = e.mean_velocity_series()
    t3 = time.perf_counter()
    e.snapshot32(out_x=outx, out_v=outv)
    t4 = time.perf_counter()
    lib = nasch._lib()
    lib.nasch_sim_state32(e._h, nasch._u32p(outx), None, N)  # positions only
    t5 = time.perf_counter()
    lib.nasch_sim_state32(e._h, None, nasch._u32p(outv), N)  # velocities only
    t6 = time.perf_counter()
    print(f"set_state32 {1e3*(t1-t0):.2f} ms, advance(20) {1e3*(t2-t1):.2f}, series {1e3*(t3-t2):.2f}, "
          f"state32 {1e3*(t4-t3):.2f}, positions only {1e3*(t5-t4):.2f}, velocities only {1e3*(t6-t5):.2f}",
          flush=True)
    e = nasch.Engine(nasch.SimParams(length=L, ncars=N, vmax=5, p=0.13, steps=100, seed=3))
    e.set_checksum(False)
for rep in range(3):
    e = nasch.Engine(nasch.SimParams(length=L, ncars=N, vmax=5, p=0.13, steps=100, seed=3))
    e.set_checksum(False)
    e.advance(0)
    t0 = time.perf_counter()
    e.job32(xin, vin, 20, out_x=outx, out_v=outv)
    t1 = time.perf_counter()
    s = e.mean_velocity_series()
    t2 = time.perf_counter()
    print(f"job32(20 steps) {1e3*(t1-t0):.2f} ms, series {1e3*(t2-t1):.2f} ms -> "
          f"{N * 20 / (t2 - t0):.3e} car-updates/s", flush=True)
