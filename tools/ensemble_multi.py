"""BASELINE config 4 on N GPUs: the 4096 rings split into contiguous ranges
balanced by cars (nasch.partition_rings), one Ensemble per GPU, no
communication while stepping, one gather of the per-ring velocity totals.

  python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
      tools/ensemble_multi.py [--steps T]

Rank 0 prints one JSON line: whole-job car-updates/s over the max-over-ranks
CUDA-event time, and a checksum of the gathered totals (equal for every N).
"""
import argparse
import hashlib
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2309_14311_b200 import nasch  # noqa: E402


def c4_specs():
    dens = [5000 + (45000 * j) // 63 for j in range(64)]
    ps = [0.0, 0.1, 0.2, 0.3, 0.4, 0.5, 0.6, 0.7]
    return [(N, p, 1 + rep * 1000 + pi * 100 + j)
            for rep in range(8) for pi, p in enumerate(ps) for j, N in enumerate(dens)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=5000)
    a = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl")
    L = 10**5
    specs = c4_specs()
    lo, hi = nasch.partition_rings([s[0] for s in specs], world)[rank]
    mine = specs[lo:hi]
    ens = nasch.Ensemble([nasch.SimParams(length=L, ncars=N, vmax=5, p=p, steps=a.steps, seed=sd)
                          for N, p, sd in mine])
    for r, (N, p, sd) in enumerate(mine):
        x, v = nasch.fill_uniform_state(L, N, 0, sd)
        ens.set_state(r, x, v)
    s = torch.cuda.ExternalStream(ens.cuda_stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0.record(s)
    ens.enqueue(a.steps)
    e1.record(s)
    ens.synchronize()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    totals = ens.sumv_totals()
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        parts = [None] * world
        dist.all_gather_object(parts, (lo, totals.tolist()))
        totals = np.array([v for _, tot in sorted(parts) for v in tot], dtype=np.uint64)
    if rank == 0:
        cars = sum(N for N, _, _ in specs)
        print(json.dumps({"metric": "car-updates/s", "config": "C4", "n_gpus": world, "steps": a.steps,
                          "value": cars * a.steps / (ms / 1e3), "ms": ms,
                          "totals_sha256": hashlib.sha256(totals.tobytes()).hexdigest()}), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
