"""Driver for timing / ncu captures of the ensemble kernel on BASELINE C4
(4096 rings of L=1e5, densities 0.05..0.5, p in {0..0.7}, 8 seeds).

  python tools/profile_c4.py [--steps S]
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2309_14311_b200 import nasch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=200)
    a = ap.parse_args()
    L = 10**5
    dens = [5000 + (45000 * j) // 63 for j in range(64)]
    ps = [0.0, 0.1, 0.2, 0.3, 0.4, 0.5, 0.6, 0.7]
    specs = [(N, p, 1 + rep * 1000 + pi * 100 + j) for rep in range(8) for pi, p in enumerate(ps)
             for j, N in enumerate(dens)]
    ens = nasch.Ensemble([nasch.SimParams(length=L, ncars=N, vmax=5, p=p, steps=a.steps, seed=sd)
                          for N, p, sd in specs])
    for r, (N, p, sd) in enumerate(specs):
        x, v = nasch.fill_uniform_state(L, N, 0, sd)
        ens.set_state(r, x, v)
    t0 = time.perf_counter()
    ens.advance(a.steps)
    t1 = time.perf_counter()
    cars = sum(N for N, _, _ in specs)
    print(f"steps={a.steps} wall_s={t1 - t0:.4f} rate={cars * a.steps / (t1 - t0):.3e}")


if __name__ == "__main__":
    main()
