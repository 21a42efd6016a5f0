"""Per-launch cost of the segmented ring's exchange, on ONE GPU.

  python tools/xchg_overhead.py [--n 200000000] [--steps 512] [--out profiles/r01_xchg_overhead.json]

The C3 ring (or --n cars at density 0.2) is split into G segments held by
this process -- all on the one visible GPU, each on its own stream -- and
advanced with each exchange mode:
  collective: step kernel, pack kernel, G*G peer copies, plan kernel
  p2p       : step kernel whose last block stores the record into every
              segment's HBM and raises flags, plan kernel that awaits them
Segments of one process are also ordered by events (no kernel ever waits
on a kernel that might not run), so on one GPU this measures the launch
and kernel overhead each mode adds per K-step launch -- not NVLink latency,
which needs two GPUs.  Wall clock around advance() (host enqueue included;
the shards' streams are synchronised at the end), min of 3.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2309_14311_b200 import nasch  # noqa: E402


def run(N, L, T, G, mode, x, v):
    os.environ["NASCH_B200_XCHG"] = mode
    prm = nasch.SimParams(length=L, ncars=N, vmax=5, p=0.13, steps=64 + 4 * T, seed=3)
    e = nasch.Engine(prm, G, nasch.Engine.CUDA)
    e.set_checksum(False)
    e.set_state(x, v)
    got_mode = e.exchange_mode
    e.advance(64)
    best = None
    for _ in range(3):
        t0 = time.perf_counter()
        e.advance(T)
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    launches = e.kernel_launches
    e.close()
    return dict(G=G, mode=mode, exchange_mode=got_mode, seconds=best,
                car_updates_per_s=N * T / best, launches_total=launches)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=200_000_000)
    ap.add_argument("--steps", type=int, default=512)
    ap.add_argument("--gs", default="1,2,4,8")
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    N, L, T = a.n, a.n * 5, a.steps
    x, v = nasch.fill_uniform_state(L, N, 0, 3)
    rows = []
    for G in [int(g) for g in a.gs.split(",")]:
        for mode in (["single"] if G == 1 else ["collective", "p2p"]):
            r = run(N, L, T, G, "collective" if mode == "single" else mode, x, v)
            r["mode"] = mode
            launches = T / 16
            r["us_per_launch"] = r["seconds"] / launches * 1e6
            rows.append(r)
            print(json.dumps(r), flush=True)
    base = rows[0]["us_per_launch"]
    for r in rows:
        r["overhead_us_per_launch_vs_one_segment"] = r["us_per_launch"] - base
    res = dict(gpu="1 B200", N=N, L=L, steps=T, K=16, rows=rows,
               note="all segments on ONE GPU (in-process, event-ordered); isolates the "
                    "exchange's launch/kernel overhead, not NVLink latency")
    if a.out:
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
