"""car-updates/s against ring size across the medium- and large-ring engines
(distributed-resident / temporal-blocked block tiles / warp tiles), density
0.2, p = 0.13, checksum off."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

from bench_configs import ev_time  # noqa: E402
from paper_2309_14311_b200 import nasch  # noqa: E402

for N in [100000, 200000, 400000, 550000, 600000, 800000, 1000000, 2000000, 4000000, 10000000, 30000000]:
    L = 5 * N
    T = max(256, min(4096, int(2e9 / N) // 32 * 32))
    x, v = nasch.fill_uniform_state(L, N, 0, 42)
    best = None
    for rep in range(3):
        e = nasch.Engine(nasch.SimParams(length=L, ncars=N, vmax=5, p=0.13, steps=T + 128, seed=42))
        e.set_checksum(False)
        e.set_state(x, v)
        e.advance(128)
        secs = ev_time(e.cuda_stream, lambda: (e.enqueue(T), e.synchronize()))
        best = secs if best is None else min(best, secs)
        spl = e.steps_per_launch
        e.close()
    print(json.dumps({"N": N, "steps": T, "us_per_step": round(1e6 * best / T, 2), "car_updates_per_s": N * T / best,
                      "steps_per_launch": spl}), flush=True)
