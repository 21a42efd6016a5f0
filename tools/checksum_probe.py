"""Checksum-on step time (the reference's stock semantics: every step's
rank-ordered row folded into FNV-1a) on one GPU:
    python tools/checksum_probe.py [L] [N] [steps]
Prints ms per step (wall clock around advance, synchronous) and the digest."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2309_14311_b200 import nasch  # noqa: E402

L = int(float(sys.argv[1])) if len(sys.argv) > 1 else 10**9
N = int(float(sys.argv[2])) if len(sys.argv) > 2 else 2 * 10**8
T = int(sys.argv[3]) if len(sys.argv) > 3 else 20
x, v = nasch.fill_uniform_state(L, N, 0, 3)
e = nasch.Engine(nasch.SimParams(length=L, ncars=N, vmax=5, p=0.13, steps=T + 3, seed=3))
e.set_checksum(True)
e.set_state(x, v)
e.advance(3)
t0 = time.perf_counter()
e.advance(T)
dt = time.perf_counter() - t0
print(f"L={L} N={N} steps={T}: {1e3 * dt / T:.3f} ms/step, {N * T / dt:.3e} car-updates/s, "
      f"checksum {e.checksum:#x}, launches {e.kernel_launches}")
