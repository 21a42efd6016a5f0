"""Small rings with the trajectory checksum on (the reference's stock
semantics): wall time of the whole run through the C ABI.
    python tools/small_checksum_probe.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2309_14311_b200 import nasch  # noqa: E402

for (L, N, T) in [(1000, 200, 1000), (10**5, 20000, 1000), (10**6, 2 * 10**5, 1000)]:
    x, v = nasch.fill_uniform_state(L, N, 0, 42)
    for ck in (False, True):
        e = nasch.Engine(nasch.SimParams(length=L, ncars=N, vmax=5, p=0.13, steps=T + 10, seed=42))
        e.set_checksum(ck)
        e.set_state(x, v)
        e.advance(10)
        t0 = time.perf_counter()
        e.advance(T)
        dt = time.perf_counter() - t0
        print(f"L={L} N={N} T={T} checksum={ck}: {1e3 * dt:.2f} ms, {N * T / dt:.3e} car-updates/s, "
              f"{1e6 * dt / T:.1f} us/step", flush=True)
