"""Frame recording cost (output = ascii / pgm) on small and medium rings."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2309_14311_b200 import nasch
for (L, N, T, stride) in [(1000, 200, 1000, 1), (1000, 200, 1000, 10), (10**6, 2*10**5, 200, 1)]:
    for mode in ("ascii", "pgm"):
        p = nasch.SimParams(length=L, ncars=N, vmax=5, p=0.13, steps=T, seed=42, output=mode, stride=stride)
        e = nasch.Engine(p)
        e.set_checksum(False)
        t0 = time.perf_counter(); e.run(); dt = time.perf_counter() - t0
        print(f"L={L} N={N} T={T} {mode} stride={stride}: {1e3*dt:.1f} ms ({1e6*dt/T:.1f} us/step), frames {e.frame_count}")
