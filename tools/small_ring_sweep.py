"""Step time against ring size across the small- and medium-ring engines
(one-warp / four-warp / one-CTA / distributed-resident), density 0.2,
p = 0.13, checksum off: ns per step and car-updates/s."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

from bench_configs import ev_time  # noqa: E402
from paper_2309_14311_b200 import nasch  # noqa: E402

T = 2000
for N in [100, 200, 400, 512, 600, 1000, 2000, 3000, 4096, 4200, 6000, 10000, 20000, 50000]:
    L = 5 * N
    x, v = nasch.fill_uniform_state(L, N, 0, 42)
    best = None
    for rep in range(3):
        e = nasch.Engine(nasch.SimParams(length=L, ncars=N, vmax=5, p=0.13, steps=T + 100, seed=42))
        e.set_checksum(False)
        e.set_state(x, v)
        e.advance(100)
        secs = ev_time(e.cuda_stream, lambda: (e.enqueue(T), e.synchronize()))
        best = secs if best is None else min(best, secs)
        e.close()
    print(json.dumps({"N": N, "ns_per_step": round(1e9 * best / T, 1), "car_updates_per_s": N * T / best}), flush=True)
