"""One grid-engine run for ncu captures: L=1e8, N=2e7, p=0.13, 12 steps."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2309_14311_b200 import nasch  # noqa: E402

L, N = 10**8, int(sys.argv[1]) if len(sys.argv) > 1 else 2 * 10**7
p = float(sys.argv[2]) if len(sys.argv) > 2 else 0.13
x, v = nasch.fill_uniform_state(L, N, 5, 3)
e = nasch.Engine(nasch.SimParams(length=L, ncars=N, vmax=5, p=p, steps=12, seed=3), 1,
                 nasch.Engine.GRID_REFERENCE)
e.set_checksum(False)
e.set_state(x, v)
e.advance(12)
print("ok", e.sumv_series()[-1])
