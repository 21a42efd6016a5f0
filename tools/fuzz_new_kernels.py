"""Randomised parity fuzz of the round-2 kernels (one GPU):
  * bit-plane grid (every WPT) vs the oracle on random rings with L % 32 == 0
    (random N, vmax <= 7, p, steps, injected velocities, a mid-run state read);
  * four-warp small-ring kernel (NASCH_B200_QUADRING=2) vs the oracle on random
    rings of 65..512 cars (u8 and u32 velocities, checksum on).
    python tools/fuzz_new_kernels.py [seconds] [seed]"""
import os
import random
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle as O  # noqa: E402
from paper_2309_14311_b200 import nasch  # noqa: E402

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
rd = random.Random(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
port = O.Port()
GRID = nasch.Engine.GRID_REFERENCE
t_end = time.time() + budget
ngrid = nquad = nmid = nq = 0


def compare(e, o, what):
    x, v = e.snapshot()
    ok = ((x == o["x"]).all() and (v == o["v"]).all() and (e.sumv_series() == o["sumv"]).all()
          and (e.wrap_series() == o["wraps"]).all() and e.checksum == o["checksum"])
    if not ok:
        print("MISMATCH", what, flush=True)
        sys.exit(1)


while time.time() < t_end:
    # grid, bit planes
    wpt = rd.choice(["1", "2", "4"])
    os.environ["NASCH_B200_GRID_WPT"] = wpt
    words = rd.choice([1, 2, 3, rd.randrange(1, 40), 256 * int(wpt) + rd.randrange(-2, 3),
                       2 * 256 * int(wpt) + rd.randrange(0, 5), rd.randrange(1, 3000)])
    L = 32 * max(1, words)
    N = max(1, min(L, int(L * rd.choice([0.02, 0.2, 0.5, 0.9, 1.0]) * rd.random() * 1.2) or 1))
    vmax = rd.randrange(1, 8)
    p = rd.choice([0.0, 1.0, rd.random()])
    T = rd.randrange(1, 80)
    seed = rd.getrandbits(63)
    x0, v0 = port.fill_uniform_state(L, N, rd.randrange(0, vmax + 1), rd.getrandbits(32))
    x0, v0 = np.asarray(x0, np.uint64), np.asarray(v0, np.uint64)
    o = port.run(L, vmax, p, seed, T, x0, v0)
    g = nasch.Engine(nasch.SimParams(length=L, ncars=N, vmax=vmax, p=p, steps=T, seed=seed), 1, GRID)
    g.set_state(x0, v0)
    g.advance(rd.randrange(0, T + 1))
    g.snapshot()
    g.advance(T)
    compare(g, o, ("grid", wpt, L, N, vmax, p, T, seed))
    g.close()
    ngrid += 1
    # four-warp small rings
    os.environ["NASCH_B200_QUADRING"] = "2"
    N = rd.randrange(65, 513)
    L = N + rd.randrange(0, 6 * N)
    vmax = rd.choice([1, 3, 5, 9, 300])
    p = rd.choice([0.0, 1.0, rd.random()])
    T = rd.randrange(1, 400)
    seed = rd.getrandbits(63)
    x0, v0 = port.fill_uniform_state(L, N, min(vmax, L - 1, rd.randrange(0, 6)), rd.getrandbits(32))
    x0, v0 = np.asarray(x0, np.uint64), np.asarray(v0, np.uint64)
    o = port.run(L, vmax, p, seed, T, x0, v0)
    e = nasch.Engine(nasch.SimParams(length=L, ncars=N, vmax=vmax, p=p, steps=T, seed=seed))
    e.set_state(x0, v0)
    k = rd.randrange(0, T + 1)
    e.advance(k)
    e.advance(T - k)
    compare(e, o, ("quad", L, N, vmax, p, T, seed))
    e.close()
    nquad += 1
    # 513..4096 cars: the distributed-resident kernel (one-CTA kernel where it does not apply)
    os.environ.pop("NASCH_B200_QUADRING", None)
    if ngrid % 8 == 0:
        N = rd.randrange(513, 4097)
        L = N + rd.randrange(0, 5 * N)
        vmax = rd.choice([1, 3, 5, 7, 300])
        p = rd.choice([0.0, 1.0, rd.random()])
        T = rd.randrange(1, 200)
        seed = rd.getrandbits(63)
        x0, v0 = port.fill_uniform_state(L, N, min(vmax, L - 1, rd.randrange(0, 6)), rd.getrandbits(32))
        x0, v0 = np.asarray(x0, np.uint64), np.asarray(v0, np.uint64)
        o = port.run(L, vmax, p, seed, T, x0, v0)
        e = nasch.Engine(nasch.SimParams(length=L, ncars=N, vmax=vmax, p=p, steps=T, seed=seed))
        e.set_state(x0, v0)
        k = rd.randrange(0, T + 1)
        e.advance(k)
        e.advance(T - k)
        compare(e, o, ("mid", L, N, vmax, p, T, seed))
        e.close()
        nmid += 1
    # the distributed-resident kernel at 20 / 24 / 32 cars per thread (QDRAW), forced on medium rings
    if ngrid % 16 == 0:
        os.environ["NASCH_B200_DR_GEOM"] = rd.choice(["3", "4", "5"])
        N = rd.randrange(4200, 60000)
        L = N + rd.randrange(0, 5 * N)
        vmax = rd.choice([1, 3, 5, 7])
        p = rd.choice([0.0, 1.0, rd.random()])
        T = rd.randrange(1, 120)
        seed = rd.getrandbits(63)
        x0, v0 = port.fill_uniform_state(L, N, min(vmax, L - 1, rd.randrange(0, 6)), rd.getrandbits(32))
        x0, v0 = np.asarray(x0, np.uint64), np.asarray(v0, np.uint64)
        o = port.run(L, vmax, p, seed, T, x0, v0)
        e = nasch.Engine(nasch.SimParams(length=L, ncars=N, vmax=vmax, p=p, steps=T, seed=seed))
        e.set_state(x0, v0)
        k = rd.randrange(0, T + 1)
        e.advance(k)
        e.advance(T - k)
        compare(e, o, ("qdraw", os.environ["NASCH_B200_DR_GEOM"], L, N, vmax, p, T, seed))
        e.close()
        os.environ.pop("NASCH_B200_DR_GEOM", None)
        nq += 1
print(f"fuzz ok: {nq} QDRAW rings, {ngrid} grid cases, {nquad} four-warp cases, {nmid} rings of 513..4096 cars", flush=True)
