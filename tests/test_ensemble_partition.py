"""Ensemble sharding across ranks: contiguous ring
ranges balanced by cars, no communication while stepping, one gather of the
per-ring totals.  The partition is checked directly, and the rank protocol
runs as world_size-2 and -3 gloo groups on CPU with the oracle standing in
for each rank's GPU ensemble (tools/ensemble_multi.py is the GPU driver)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2309_14311_b200 import nasch


def test_partition_covers_and_balances():
    rng = np.random.default_rng(5)
    for world in (1, 2, 3, 4, 8):
        for n in ([5000 + (45000 * j) // 63 for j in range(64)] * 8, list(rng.integers(1, 90000, 500)), [7] * 3):
            parts = nasch.partition_rings(n, world)
            assert len(parts) == world
            assert parts[0][0] == 0 and parts[-1][1] == len(n)
            assert all(parts[i][1] == parts[i + 1][0] for i in range(world - 1))
            loads = [sum(n[a:b]) for a, b in parts]
            if len(n) >= 4 * world:
                assert max(loads) <= sum(n) / world + max(n)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, specs, out):
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
    import oracle
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    port_impl = oracle.Port()
    lo, hi = nasch.partition_rings([s[1] for s in specs], world)[rank]
    totals = []
    for (L, N, vmax, p, T, seed) in specs[lo:hi]:
        x0, v0 = port_impl.init_state(L, N)
        o = port_impl.run(L, vmax, p, seed, T, x0, v0, want_checksum=False)
        totals.append(int(o["sumv"].sum()))
    parts = [None] * world
    dist.all_gather_object(parts, (lo, totals))
    if rank == 0:
        out.put([v for _, tot in sorted(parts) for v in tot])
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_partitioned_ensemble_gloo(port, world):
    rng = np.random.default_rng(world)
    specs = [(int(L), int(rng.integers(1, L // 2)), 5, float(rng.choice([0.1, 0.3, 0.6])), 30,
              int(rng.integers(0, 2**30))) for L in rng.integers(50, 4000, 17)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    prt = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, prt, specs, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    got = q.get(timeout=600)
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    want = []
    for (L, N, vmax, p, T, seed) in specs:
        x0, v0 = port.init_state(L, N)
        want.append(int(port.run(L, vmax, p, seed, T, x0, v0, want_checksum=False)["sumv"].sum()))
    assert got == want
