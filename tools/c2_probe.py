"""BASELINE config 2 (L=1e6, N=2e5, p=0.25, v uniform in [0,5]) on the
distributed-resident engine, for ncu captures and timing:
    python tools/c2_probe.py [steps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2309_14311_b200 import nasch  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
L, N = 10**6, 2 * 10**5
x, v = nasch.fill_uniform_state(L, N, 5, 2)
e = nasch.Engine(nasch.SimParams(length=L, ncars=N, vmax=5, p=0.25, steps=T + 1000, seed=2))
e.set_checksum(False)
e.set_state(x, v)
e.advance(1000)
t0 = time.perf_counter()
e.advance(T)
dt = time.perf_counter() - t0
print(f"C2 {T} steps: {1e3 * dt:.2f} ms, {N * T / dt:.3e} car-updates/s, launches {e.kernel_launches}")
