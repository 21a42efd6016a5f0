"""Per-launch time of the temporal-blocked step kernel against its depth K
on BASELINE config 3 (L=1e9, N=2e8): time(K) = a + b*K separates the
per-launch fixed cost (state load/store not hidden by compute, wave tail,
plan) from the per-step compute.  Also times the checksum-on path (one
step per launch + the on-device FNV fold of the whole rank-ordered row).

  python tools/tb_k_sweep.py [--ks 1,2,4,8,12,16] [--launches 12] [--checksum-steps 4]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2309_14311_b200 import nasch  # noqa: E402

L, N, P, SEED = 10**9, 2 * 10**8, 0.13, 3


def per_launch_ms(e, k, launches):
    s = torch.cuda.ExternalStream(e.cuda_stream)
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(launches + 1)]
    torch.cuda.synchronize()
    evs[0].record(s)
    for i in range(launches):
        e.enqueue(k)
        evs[i + 1].record(s)
    e.synchronize()
    torch.cuda.synchronize()
    return [evs[i].elapsed_time(evs[i + 1]) for i in range(launches)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ks", default="1,2,4,8,12,16")
    ap.add_argument("--launches", type=int, default=12)
    ap.add_argument("--checksum-steps", type=int, default=4)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    x, v = nasch.fill_uniform_state(L, N, 0, SEED)
    res = {"L": L, "N": N, "k": {}}
    for k in [int(t) for t in a.ks.split(",")]:
        os.environ["NASCH_B200_K"] = str(max(k, 2))
        e = nasch.Engine(nasch.SimParams(length=L, ncars=N, vmax=5, p=P, steps=10**6, seed=SEED))
        e.set_checksum(False)
        e.set_state(x, v)
        e.advance(256)
        ms = per_launch_ms(e, k, a.launches)
        med = float(np.median(ms[2:]))
        res["k"][k] = {"spl": e.steps_per_launch, "launch_ms_median": med, "ms_per_step": med / k,
                       "car_updates_per_s": N * k / (med / 1e3), "launch_ms": ms}
        print(json.dumps({"k": k, **{kk: vv for kk, vv in res["k"][k].items() if kk != "launch_ms"}}),
              flush=True)
        e.close()
    ks = sorted(res["k"])
    if len(ks) >= 2:
        A = np.array([[1.0, k] for k in ks])
        y = np.array([res["k"][k]["launch_ms_median"] for k in ks])
        coef, *_ = np.linalg.lstsq(A, y, rcond=None)
        res["fit"] = {"a_ms_per_launch": float(coef[0]), "b_ms_per_step": float(coef[1])}
        print(json.dumps(res["fit"]), flush=True)
    os.environ.pop("NASCH_B200_K", None)
    if a.checksum_steps:
        e = nasch.Engine(nasch.SimParams(length=L, ncars=N, vmax=5, p=P, steps=10**6, seed=SEED))
        e.set_checksum(True)
        e.set_state(x, v)
        e.advance(1)
        ms = per_launch_ms(e, 1, a.checksum_steps)
        res["checksum_on"] = {"ms_per_step": float(np.median(ms)), "all_ms": ms,
                              "car_updates_per_s": N / (float(np.median(ms)) / 1e3)}
        print(json.dumps({"checksum_on": res["checksum_on"]}), flush=True)
        e.close()
    if a.out:
        with open(a.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
