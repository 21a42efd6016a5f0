"""BASELINE config 1 (L=1000, N=200, 1000 steps) and other small rings: step
time of the four-warp register kernel against the one-warp kernel
(NASCH_B200_QUADRING=0), CUDA-event time of one resident launch, checksum off."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

from bench_configs import ev_time  # noqa: E402
from paper_2309_14311_b200 import nasch  # noqa: E402


def one(L, N, p, T, quad):
    os.environ["NASCH_B200_QUADRING"] = "1" if quad else "0"
    x, v = nasch.fill_uniform_state(L, N, 0, 42)
    best = None
    for rep in range(5):
        e = nasch.Engine(nasch.SimParams(length=L, ncars=N, vmax=5, p=p, steps=T + 100, seed=42))
        e.set_checksum(False)
        e.set_state(x, v)
        e.advance(100)
        secs = ev_time(e.cuda_stream, lambda: (e.enqueue(T), e.synchronize()))
        best = secs if best is None else min(best, secs)
        xs, vs = e.snapshot()
        s = e.sumv_series()
        e.close()
    return best, xs, vs, s


for (L, N, p, T) in [(1000, 200, 0.13, 1000), (1000, 203, 0.13, 1000), (500, 100, 0.2, 1000), (2500, 500, 0.13, 1000),
                     (2500, 509, 0.3, 1000)]:
    tq, xq, vq, sq = one(L, N, p, T, True)
    tw, xw, vw, sw = one(L, N, p, T, False)
    print(json.dumps({"L": L, "N": N, "steps": T, "quad_ns_per_step": 1e9 * tq / T, "warp_ns_per_step": 1e9 * tw / T,
                      "quad_car_updates_per_s": N * T / tq, "warp_car_updates_per_s": N * T / tw,
                      "equal": bool((xq == xw).all() and (vq == vw).all() and (sq == sw).all())}), flush=True)
