import os, sys
sys.path.insert(0, "/root/repo")
from paper_2309_14311_b200 import nasch
L, N = 10**9, 2*10**8
x, v = nasch.fill_uniform_state(L, N, 0, 3)
e = nasch.Engine(nasch.SimParams(length=L, ncars=N, vmax=5, p=0.13, steps=100, seed=3))
e.set_checksum(True)
e.set_state(x, v)
e.advance(3)
print("ok", e.checksum)
