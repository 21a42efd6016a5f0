"""Epoch timeline of the distributed-resident kernel (diagnostic build).

  make -C paper_2309_14311_b200/csrc OUT=$PWD/tools/_variants/drtrace.so \
       BUILD=/tmp/vdt/ CLI=/tmp/vdt/nasch NVCC="nvcc -DNB_DR_TRACE"
  NASCH_B200_LIB=tools/_variants/drtrace.so python tools/dr_trace.py [--L .. --N ..]

Prints, per epoch, the %globaltimer offsets (ns) of: worker 0 ready (plan
and halo in hand), worker 0 finished its steps, worker 0 signalled, the last
worker signalled, the planner saw every worker's S_e, finished the cone, and
published plan(e+1).
"""
import argparse
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2309_14311_b200 import capi, nasch  # noqa: E402

NAMES = ["w0_ready", "w0_steps", "w0_sig", "wlast_sig", "pl_all", "pl_cone", "-", "pl_pub"]


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
    ne = min(256, (a.steps + 31) // 32)
    t0 = t[0, 0] if t[0, 0] else t[0, 1]
    print("epoch " + " ".join(f"{n:>10s}" for n in NAMES))
    for i in range(min(ne, 12)):
        print(f"{i:5d} " + " ".join(f"{(x - t0) if x else -1:10d}" for x in t[i]))
    d = np.diff(t[1:ne - 1, 0])
    print("epoch period ns: median", int(np.median(d)))
    for a_, b_ in [(0, 1), (1, 2), (2, 3), (4, 5), (5, 7)]:
        seg = t[1:ne - 1, b_] - t[1:ne - 1, a_]
        print(f"{NAMES[a_]:>10s} -> {NAMES[b_]:<10s} median {int(np.median(seg)):8d} ns")
    seg = t[2:ne - 1, 0] - t[1:ne - 2, 7]
    print(f"{'pl_pub(e)':>10s} -> {'w0_ready(e+1)':<12s} median {int(np.median(seg)):8d} ns")
    seg = t[2:ne - 1, 4] - t[1:ne - 2, 3]
    print(f"{'wlast_sig(e)':>10s} -> {'pl_all(e+1)':<12s} median {int(np.median(seg)):8d} ns")
    cc = (ctypes.c_ulonglong * 2)()
    if lib.nasch_b200_cone_cycles(cc) == 0 and cc[1]:
        print(f"planner cone loop: {cc[0] / cc[1]:.0f} cycles per cone step ({cc[1]} steps)")
    wb = (ctypes.c_ulonglong * (64 * 160 * 4))()
    assert lib.nasch_b200_dr_wtrace(wb, 64 * 160 * 4) == 0
    w = np.frombuffer(wb, dtype=np.uint64).reshape(64, 160, 4).astype(np.int64)
    G = int((w[1, :, 3] > 0).sum())
    ready = w[2:min(ne, 64) - 1, :G, 0]
    sig = w[2:min(ne, 64) - 1, :G, 3]
    for a_, b_, nm in [(0, 1, "steps"), (1, 2, "-"), (2, 3, "mailbox+store+reduce+signal")]:
        seg = w[2:min(ne, 64) - 1, :G, b_] - w[2:min(ne, 64) - 1, :G, a_]
        print(f"worker {nm:>20s}: median {int(np.median(seg))} ns  p90 {int(np.percentile(seg, 90))}")
    busy = sig - ready
    late = sig - sig.min(axis=1, keepdims=True)
    print(f"workers {G}: ready->signal median {int(np.median(busy))} ns, p90 {int(np.percentile(busy, 90))}, max {int(busy.max())}")
    print("slowest workers (median ready->signal):", sorted(((int(np.median(busy[:, g])), g) for g in range(G)))[-6:])
    print("ready spread per epoch (max-min) median:", int(np.median(ready.max(1) - ready.min(1))))
    print("signal spread per epoch (max-min) median:", int(np.median(late.max(1))))


if __name__ == "__main__":
    main()
