"""The multi-GPU segmented-ring protocol, run as world_size-2 (and 3)
torch.distributed gloo process groups on CPU and checked bit-exactly
against the single-ring oracle.  The GPU implementation
(csrc/sharded.cu, shard_kernels.cuh) moves exactly these records; its own
bit-exactness for G shards is tested in tests/test_gpu_sharded.py."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import shard_protocol as sp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, cfg, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    L, N, vmax, p, seed, K, launches, x0, v0 = cfg
    sh = sp.Shard(L, N, vmax, p, seed, world, rank, x0, v0, K)
    for _ in range(launches):
        recs = [None] * world
        dist.all_gather_object(recs, sh.pack())
        Ws, cs = sh.plan(recs)
        sh.advance(Ws, cs)
    seg = [None] * world
    dist.all_gather_object(seg, (sh.ids[0], sh.x, sh.v, sh.sumv, sh.W))
    if rank == 0:
        out.put(seg)
    dist.barrier()
    dist.destroy_process_group()


def _run(world, cfg):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    seg = q.get(timeout=600)
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    return seg


@pytest.mark.parametrize("world,K,vmax,p", [(2, 4, 5, 0.3), (3, 6, 3, 0.6)])
def test_protocol_gloo_matches_oracle(port, world, K, vmax, p):
    L, N, seed, launches = 3000, 700, 17, 6
    rng = np.random.default_rng(world)
    x0 = np.sort(rng.choice(L, N, replace=False)).astype(np.uint64)
    v0 = rng.integers(0, vmax + 1, N).astype(np.uint64)
    seg = _run(world, (L, N, vmax, p, seed, K, launches, [int(a) for a in x0], [int(a) for a in v0]))
    x_id = sum((s[1] for s in seg), [])
    v_id = sum((s[2] for s in seg), [])
    W = seg[0][4]
    assert all(s[4] == W for s in seg)  # replicated rank offset
    sumv = np.sum([s[3] for s in seg], axis=0)
    T = K * launches
    o = port.run(L, vmax, p, seed, T, x0, v0, want_checksum=False)
    xr, vr = sp.rank_order(x_id, v_id, W, N)
    assert xr == [int(a) for a in o["x"]]
    assert vr == [int(a) for a in o["v"]]
    assert [int(a) for a in sumv] == [int(a) for a in o["sumv"]]
