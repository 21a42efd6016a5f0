import json, os, sys
ROOT = os.getcwd()
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tools"))
from bench_configs import ev_time
from paper_2309_14311_b200 import nasch
for N in [600000, 1000000, 2000000, 4000000]:
    L = 5 * N
    T = max(256, min(4096, int(2e9 / N) // 32 * 32))
    x, v = nasch.fill_uniform_state(L, N, 0, 42)
    for tile in ["medium", "large"]:
        for waves in ["", "1", "2", "4"]:
            os.environ["NASCH_B200_TILE"] = tile
            if waves: os.environ["NASCH_B200_WAVES"] = waves
            else: os.environ.pop("NASCH_B200_WAVES", None)
            best = None
            for rep in range(3):
                e = nasch.Engine(nasch.SimParams(length=L, ncars=N, vmax=5, p=0.13, steps=T + 128, seed=42))
                e.set_checksum(False); e.set_state(x, v); e.advance(128)
                secs = ev_time(e.cuda_stream, lambda: (e.enqueue(T), e.synchronize()))
                best = secs if best is None else min(best, secs)
                e.close()
            print(N, tile, "waves", waves or "default", round(1e6 * best / T, 2), "us/step", "%.3g" % (N * T / best), flush=True)
