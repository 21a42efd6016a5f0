"""A/B of the grid engine's bit-plane and byte-per-cell forms (one GPU):
us per step at L = 1e8 for both, equality of the final states."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

from bench_configs import ev_time  # noqa: E402
from paper_2309_14311_b200 import nasch  # noqa: E402


def one(L, N, p, T, seed, force_bytes):
    if force_bytes:
        os.environ["NASCH_B200_GRID_BYTES"] = "1"
    else:
        os.environ.pop("NASCH_B200_GRID_BYTES", None)
    x, v = nasch.fill_uniform_state(L, N, 5, seed)
    e = nasch.Engine(nasch.SimParams(length=L, ncars=N, vmax=5, p=p, steps=T + 8, seed=seed), 1,
                     nasch.Engine.GRID_REFERENCE)
    e.set_checksum(False)
    e.set_state(x, v)
    e.advance(8)
    secs = ev_time(e.cuda_stream, lambda: (e.enqueue(T), e.synchronize()))
    xs, vs = e.snapshot()
    s = e.sumv_series()
    e.close()
    return secs / T * 1e6, xs, vs, s


for (L, N, p, T, seed) in [(10**6, 2 * 10**5, 0.25, 2000, 2), (10**8, 2 * 10**7, 0.13, 200, 3),
                           (10**8, 6 * 10**7, 0.5, 200, 5)]:
    ub, xb, vb, sb = one(L, N, p, T, seed, False)
    uy, xy, vy, sy = one(L, N, p, T, seed, True)
    print(json.dumps({"L": L, "N": N, "p": p, "us_per_step_bits": ub, "us_per_step_bytes": uy,
                      "equal": bool((xb == xy).all() and (vb == vy).all() and (sb == sy).all())}), flush=True)
