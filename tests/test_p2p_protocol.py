"""CPU model of the segmented ring's peer-memory exchange (sharded.cu
launch_p2p, shard_kernels.cuh shard_push / shard_plan_kernel), run by G
processes that share memory the way the GPUs share HBM over NVLink.

Each "shard" process owns a receive area rec[2][G][W] and flags[G].  Per
launch seq it (1) publishes its record for seq into slot [seq & 1][g] of
EVERY shard and then raises flags_h[g] = seq (the step kernel's last block),
and (2) waits until its own flags[*] >= seq and reads slot [seq & 1][*]
(the plan kernel).  The claim under test is the one the kernels rely on:
two slots suffice -- no record is overwritten while a slower shard still
reads it -- for any relative speed of the shards.  Random delays are put
between every publish and inside every read, and each word carries
(seq, source) so a torn or overwritten record is detected.

This is test infrastructure: it restates the protocol, it does not run the
CUDA kernels (those are covered by tests/test_gpu_sharded.py)."""
import multiprocessing as mp
import random
import time

import numpy as np
import pytest

W = 24  # words per record (the real record is 544 u32)


def _shard(g, G, launches, seed, shm_names, out):
    from multiprocessing import shared_memory

    shms = [shared_memory.SharedMemory(name=n) for n in shm_names]
    areas = [np.ndarray((G + 2 * G * W,), np.int64, buffer=s.buf) for s in shms]
    rng = random.Random(seed * 131 + g)
    bad = 0
    try:
        for seq in range(1, launches + 1):
            time.sleep(rng.random() * 2e-4)  # the step kernel's duration varies per shard
            slot = (seq & 1) * G + g
            word = seq * 1000 + g
            for h in range(G):  # shard_push: record into every shard, then the flags
                areas[h][G + slot * W:G + (slot + 1) * W] = word
            for h in range(G):
                areas[h][g] = seq
            deadline = time.time() + 30
            while (areas[g][:G] < seq).any():  # shard_plan_kernel: wait for every record seq
                if time.time() > deadline:
                    out.put((g, "timeout", seq))
                    return
            for src in range(G):
                base = G + ((seq & 1) * G + src) * W
                first = int(areas[g][base])
                if rng.random() < 0.3:
                    time.sleep(rng.random() * 3e-4)  # a slow reader
                last = int(areas[g][base + W - 1])
                if first != seq * 1000 + src or last != first:
                    bad += 1
        out.put((g, "ok", bad))
    finally:
        for s in shms:
            s.close()


@pytest.mark.parametrize("G", [2, 3, 5])
def test_two_slots_suffice_under_skew(G):
    from multiprocessing import shared_memory

    ctx = mp.get_context("spawn")
    shms = [shared_memory.SharedMemory(create=True, size=8 * (G + 2 * G * W)) for _ in range(G)]
    try:
        for s in shms:
            np.ndarray((G + 2 * G * W,), np.int64, buffer=s.buf)[:] = 0
        out = ctx.Queue()
        procs = [ctx.Process(target=_shard, args=(g, G, 150, G, [s.name for s in shms], out))
                 for g in range(G)]
        for p in procs:
            p.start()
        res = [out.get(timeout=120) for _ in range(G)]
        for p in procs:
            p.join(timeout=60)
        assert all(r[1] == "ok" for r in res), res
        assert sum(r[2] for r in res) == 0, res
    finally:
        for s in shms:
            s.close()
            s.unlink()
