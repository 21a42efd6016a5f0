"""Throughput of the cell-array engine (NASCH_ENGINE_GRID_REFERENCE on the
GPU, csrc/grid.cu) against its HBM roofline, one GPU.

  python tools/grid_bench.py [--out profiles/r01_grid.json]

One step reads the L cells and writes the L cells of the next array:
algorithmic bytes per step = 2 L at one byte per cell (round 1 also made a
count pass and was quoted against 3 L, reported too as hbm_frac_3L).  The
bit-plane form (csrc/grid_bits.cuh; vmax <= 7, L % 32 == 0) moves half a
byte per cell each way; its rows are still quoted against 2 L / 3 L.
CUDA-event time on the engine stream, state resident, checksum off."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))

from bench_configs import ev_time  # noqa: E402
from paper_2309_14311_b200 import nasch  # noqa: E402


def peak_gbs():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"])
    except Exception:
        return 6650.0


def one(L, N, p, T, seed):
    x, v = nasch.fill_uniform_state(L, N, 5, seed)
    prm = nasch.SimParams(length=L, ncars=N, vmax=5, p=p, steps=T + 8, seed=seed)
    e = nasch.Engine(prm, 1, nasch.Engine.GRID_REFERENCE)
    e.set_checksum(False)
    e.set_state(x, v)
    e.advance(8)
    secs = ev_time(e.cuda_stream, lambda: (e.enqueue(T), e.synchronize()))
    xs, vs = e.snapshot()
    s = e.sumv_series()
    ok = bool((xs[1:] > xs[:-1]).all() and int(vs.sum()) == int(s[-1]))
    e.close()
    gbs = 2 * L * T / secs / 1e9
    return {"L": L, "N": N, "p": p, "steps": T, "seconds": secs, "car_updates_per_s": N * T / secs,
            "cells_per_s": L * T / secs, "algorithmic_GBs": gbs, "hbm_frac": gbs / peak_gbs(),
            "hbm_frac_3L": 1.5 * gbs / peak_gbs(),
            "us_per_step": secs / T * 1e6, "invariants_ok": ok}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    rows = [one(10**6, 2 * 10**5, 0.25, 2000, 2), one(10**8, 2 * 10**7, 0.13, 200, 3),
            one(10**8, 6 * 10**7, 0.5, 200, 5)]
    for r in rows:
        print(json.dumps(r), flush=True)
    if a.out:
        with open(a.out, "w") as f:
            json.dump({"gpu": "1 B200", "peak_gbs": peak_gbs(), "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()
