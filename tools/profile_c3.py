"""Small driver for timing / ncu captures of the step kernels on C3.

  python tools/profile_c3.py [--steps S] [--warmup W] [--L ..] [--N ..]

Builds the ring (default C3: L=1e9, N=2e8, p=0.13, vmax=5, seeded uniform
init), advances W steps, then S more timed with CUDA events on the engine's
stream.  NASCH_B200_K selects the temporal-blocking depth (1 = single-step
kernel).
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
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--L", type=int, default=10**9)
    ap.add_argument("--N", type=int, default=2 * 10**8)
    ap.add_argument("--p", type=float, default=0.13)
    ap.add_argument("--events", action="store_true")
    a = ap.parse_args()
    x, v = nasch.fill_uniform_state(a.L, a.N, 0, 3)
    p = nasch.SimParams(length=a.L, ncars=a.N, vmax=5, p=a.p, steps=a.warmup + a.steps, seed=3)
    e = nasch.Engine(p)
    e.set_checksum(False)
    e.set_state(x, v)
    e.advance(a.warmup)
    ms = None
    if a.events:
        import torch
        s = torch.cuda.ExternalStream(e.cuda_stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(s)
        e.enqueue(a.steps)
        e1.record(s)
        e.synchronize()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.steps
    t0 = time.perf_counter()
    if not a.events:
        e.advance(a.steps)
    t1 = time.perf_counter()
    rate = a.N / (ms / 1e3) if ms else None
    print(f"K={e.steps_per_launch} steps={a.steps} event_ms_per_step={ms} "
          f"wall_ms_per_step={(t1 - t0) * 1e3 / a.steps:.4f} launches={e.kernel_launches} "
          f"rate={rate}")


if __name__ == "__main__":
    main()
