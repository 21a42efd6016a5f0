"""Grid engine step time with the trajectory checksum off and on (L=1e8, N=2e7)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2309_14311_b200 import nasch
L, N = 10**8, 2 * 10**7
x, v = nasch.fill_uniform_state(L, N, 5, 3)
for ck in (False, True):
    e = nasch.Engine(nasch.SimParams(length=L, ncars=N, vmax=5, p=0.13, steps=40, seed=3), 1, nasch.Engine.GRID_REFERENCE)
    e.set_checksum(ck)
    e.set_state(x, v)
    e.advance(5)
    t0 = time.perf_counter(); e.advance(20); dt = time.perf_counter() - t0
    print(f"grid L=1e8 N=2e7 checksum={ck}: {1e3*dt/20:.3f} ms/step, checksum {e.checksum:#x}")

# a small ring (C1's size): per-step launch latency
L, N = 1000, 200
x, v = nasch.fill_uniform_state(L, N, 0, 42)
for ck in (False, True):
    e = nasch.Engine(nasch.SimParams(length=L, ncars=N, vmax=5, p=0.13, steps=1010, seed=42), 1, nasch.Engine.GRID_REFERENCE)
    e.set_checksum(ck)
    e.set_state(x, v)
    e.advance(10)
    t0 = time.perf_counter(); e.advance(1000); dt = time.perf_counter() - t0
    print(f"grid L=1e3 N=200 checksum={ck}: {1e3*dt/1000:.3f} ms/step")
