"""Epoch timeline of the distributed-resident kernel (diagnostic build).

  make -C paper_2309_14311_b200/csrc OUT=$PWD/tools/_variants/drtrace.so \
       BUILD=/tmp/vdt/ CLI=/tmp/vdt/nasch NVCC="nvcc -DNB_DR_TRACE"
  NASCH_B200_LIB=tools/_variants/drtrace.so python tools/dr_trace.py [--L .. --N ..]

Prints, per epoch, the %globaltimer offsets (ns) of: worker 0 got the plan,
worker 0 finished its steps, worker 0 signalled, the last worker signalled,
the planner saw all signals, planner started / finished the cone, planner
published the next plan.
"""
import argparse
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2309_14311_b200 import capi, nasch  # noqa: E402

NAMES = ["w0_plan", "w0_steps", "w0_sig", "wlast_sig", "pl_seen", "pl_cone0", "pl_cone1", "pl_pub"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--L", type=int, default=10**6)
    ap.add_argument("--N", type=int, default=2 * 10**5)
    ap.add_argument("--p", type=float, default=0.25)
    ap.add_argument("--steps", type=int, default=320)
    a = ap.parse_args()
    x, v = nasch.fill_uniform_state(a.L, a.N, 5, 1)
    e = nasch.Engine(nasch.SimParams(length=a.L, ncars=a.N, vmax=5, p=a.p, steps=a.steps + 64, seed=1))
    e.set_checksum(False)
    e.set_state(x, v)
    e.advance(32)
    e.advance(a.steps)
    lib = capi.load()
    buf = (ctypes.c_ulonglong * (256 * 8))()
    assert lib.nasch_b200_dr_trace(buf, 256 * 8) == 0
    t = np.frombuffer(buf, dtype=np.uint64).reshape(256, 8).astype(np.int64)
    ne = min(256, (a.steps + 15) // 16)
    t0 = t[0, 0] if t[0, 0] else t[0, 1]
    print("epoch " + " ".join(f"{n:>10s}" for n in NAMES))
    for i in range(min(ne, 12)):
        print(f"{i:5d} " + " ".join(f"{(x - t0) if x else -1:10d}" for x in t[i]))
    d = np.diff(t[1:ne - 1, 0])
    print("epoch period ns: median", int(np.median(d)))
    for a_, b_ in [(0, 1), (1, 2), (2, 3), (3, 4), (4, 5), (5, 6), (6, 7)]:
        seg = t[1:ne - 1, b_] - t[1:ne - 1, a_]
        print(f"{NAMES[a_]:>10s} -> {NAMES[b_]:<10s} median {int(np.median(seg)):8d} ns")
    seg = t[2:ne - 1, 0] - t[1:ne - 2, 7]
    print(f"{'pl_pub':>10s} -> {'next w0_plan':<12s} median {int(np.median(seg)):8d} ns")


if __name__ == "__main__":
    main()
