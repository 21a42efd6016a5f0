"""GPU parity of the segmented ring (ShardedRing): G contiguous car segments
exchanging a halo and the origin-cone window once per launch must give the
single-ring trajectory bit for bit, for every G -- the B200 form of the
reference's worker-count invariance (test_engine.cpp:136-152,
test_capi.cpp:121-136).  Several shards share one GPU here (in-process
peer-copy exchange); the NCCL exchange moves the same records."""
import os

import numpy as np
import pytest

from paper_2309_14311_b200 import nasch

pytestmark = pytest.mark.gpu

CUDA = nasch.Engine.CUDA


def mk(L, N, vmax, p, steps, seed, output="none", stride=1):
    return nasch.SimParams(length=L, ncars=N, vmax=vmax, p=p, steps=steps, seed=seed,
                           output=output, stride=stride)


@pytest.fixture(params=["p2p", "collective"])
def xchg(request):
    """Both segment exchanges: records stored into peer HBM by the step
    kernel (default) and the collective path (peer copies / NCCL)."""
    old = os.environ.get("NASCH_B200_XCHG")
    os.environ["NASCH_B200_XCHG"] = request.param
    yield request.param
    if old is None:
        os.environ.pop("NASCH_B200_XCHG", None)
    else:
        os.environ["NASCH_B200_XCHG"] = old


MODE = {"p2p": 2, "collective": 1}


@pytest.fixture
def k_env():
    old = os.environ.get("NASCH_B200_K")
    yield
    if old is None:
        os.environ.pop("NASCH_B200_K", None)
    else:
        os.environ["NASCH_B200_K"] = old


def run_engine(params, workers, kind, x0=None, v0=None, steps=None, checksum=False, chunks=None):
    e = nasch.Engine(params, workers, kind)
    mode = e.exchange_mode
    e.set_checksum(checksum)
    if x0 is not None:
        e.set_state(x0, v0)
    for c in (chunks or [steps if steps is not None else params.steps]):
        e.advance(c)
    x, v = e.snapshot()
    out = dict(x=x, v=v, sumv=e.sumv_series(), wraps=e.wrap_series(), checksum=e.checksum,
               obs=e.observables(), spl=e.steps_per_launch, mode=mode)
    e.close()
    return out


@pytest.mark.parametrize("G", [2, 3, 4, 7])
def test_shards_match_oracle(port, xchg, G):
    rng = np.random.default_rng(G)
    for trial, (L, N, vmax, p) in enumerate([(40000, 6000, 5, 0.13), (9000, 8000, 5, 0.5),
                                             (3 * 10**5, 25000, 12, 0.3), (20000, 2000, 3, 0.9)]):
        x0 = np.sort(rng.choice(L, N, replace=False)).astype(np.uint64)
        v0 = rng.integers(0, min(vmax, L - 1) + 1, N).astype(np.uint64)
        T = 70
        o = port.run(L, vmax, p, 5 + trial, T, x0, v0, want_checksum=False)
        g = run_engine(mk(L, N, vmax, p, T, 5 + trial), G, CUDA, x0, v0, chunks=[13, 57])
        assert g["mode"] == MODE[xchg]
        assert (g["x"] == o["x"]).all() and (g["v"] == o["v"]).all(), (G, trial)
        assert (g["sumv"] == o["sumv"]).all()
        assert (g["wraps"] == o["wraps"]).all()


@pytest.mark.parametrize("K", [2, 5, 16])
def test_shard_depths_and_checksum(port, k_env, K):
    os.environ["NASCH_B200_K"] = str(K)
    L, N, vmax, p, T = 12000, 5000, 5, 0.35, 45
    x0, v0 = port.init_state(L, N)
    o = port.run(L, vmax, p, 21, T, x0, v0)
    g = run_engine(mk(L, N, vmax, p, T, 21), 3, CUDA, checksum=True)
    assert g["spl"] == K
    assert g["checksum"] == o["checksum"]
    assert (g["x"] == o["x"]).all() and (g["sumv"] == o["sumv"]).all()


def test_shards_equal_single_gpu_engine_long_run(xchg):
    L, N = 2 * 10**6, 4 * 10**5
    x0, v0 = nasch.fill_uniform_state(L, N, 5, 4)
    ref = run_engine(mk(L, N, 5, 0.25, 600, 8), 1, 0, x0, v0)
    for G in (2, 5):
        g = run_engine(mk(L, N, 5, 0.25, 600, 8), G, CUDA, x0, v0)
        assert (g["x"] == ref["x"]).all() and (g["v"] == ref["v"]).all()
        assert (g["sumv"] == ref["sumv"]).all() and g["obs"] == ref["obs"]


def test_shard_frames_match_single(tmp_path):
    p = mk(5000, 800, 5, 0.3, 40, 3, output="ascii", stride=7)
    a = nasch.Engine(p, 1, 0)
    a.set_checksum(False)
    a.run()
    b = nasch.Engine(p, 4, CUDA)
    b.set_checksum(False)
    b.run()
    assert a.frame_count == b.frame_count == 6
    a.write_ascii(str(tmp_path / "a.txt"))
    b.write_ascii(str(tmp_path / "b.txt"))
    assert open(tmp_path / "a.txt").read() == open(tmp_path / "b.txt").read()


def test_nccl_distributed_path_single_rank(port, xchg):
    """The one-process-per-GPU constructor with a 1-rank NCCL communicator:
    exercises libnccl loading, communicator setup, the ncclAllGather
    exchange on the real device and, for p2p, the cudaIpcMemHandle swap and
    agreement over NCCL, the push from the step kernel and the flag wait."""
    L, N, vmax, p, T = 30000, 9000, 5, 0.2, 48
    x0, v0 = nasch.fill_uniform_state(L, N, 5, 12)
    o = port.run(L, vmax, p, 4, T, x0.astype(np.uint64), v0.astype(np.uint64), want_checksum=False)
    e = nasch.Engine.distributed(mk(L, N, vmax, p, T, 4), 0, 1, nasch.nccl_unique_id())
    assert e.shard_range() == (0, N)
    assert e.exchange_mode == MODE[xchg]
    e.set_state(x0, v0)
    e.advance(T)
    x, v = e.snapshot()
    assert (x == o["x"]).all() and (v == o["v"]).all()
    assert (e.sumv_series() == o["sumv"]).all()


def test_too_small_to_shard_runs_on_one_gpu(port):
    """A ring too small to split still runs (on one GPU) with the same
    trajectory, as the reference accepts any worker count."""
    e = nasch.Engine(mk(1000, 100, 5, 0.3, 10, 1), 4, CUDA)
    e.run()
    x, v = port.init_state(1000, 100)
    o = port.run(1000, 5, 0.3, 1, 10, x, v)
    assert e.checksum == o["checksum"]
    with pytest.raises(nasch.NaschError, match="too small"):  # explicit distributed use
        nasch.Engine.distributed(mk(1000, 100, 5, 0.3, 10, 1), 0, 4, nasch.nccl_unique_id())


def test_shard_checksum_on_device_many_chunks(port, k_env):
    """The segmented ring's on-device checksum: every shard's pieces of the
    rank-ordered row span several 4096-value chunks, the rank-0 car sits
    inside a shard (its pieces split), and the composed digest equals the
    reference's serial FNV-1a at every step count."""
    os.environ.pop("NASCH_B200_K", None)
    L, N, vmax, p, T = 200000, 40000, 5, 0.3, 60
    x0, v0 = nasch.fill_uniform_state(L, N, 5, 31)
    o = port.run(L, vmax, p, 9, T, x0.astype(np.uint64), v0.astype(np.uint64))
    for G in (2, 3, 5):
        g = run_engine(mk(L, N, vmax, p, T, 9), G, CUDA, x0, v0, checksum=True, chunks=[17, T])
        assert g["checksum"] == o["checksum"], G
        assert (g["x"] == o["x"]).all()


def test_p2p_exchange_resume_and_many_launches(port, xchg):
    """set_state in the middle of a peer-exchange run (the collective
    re-initialisation, then the launch counter and slot parity carry on),
    K = 16 launches past both receive slots many times, and the result is
    the oracle's."""
    L, N, vmax, p = 60000, 12000, 5, 0.4
    x0, v0 = nasch.fill_uniform_state(L, N, 5, 17)
    x0 = x0.astype(np.uint64)
    v0 = v0.astype(np.uint64)
    o1 = port.run(L, vmax, p, 6, 37, x0, v0, want_checksum=False)
    e = nasch.Engine(mk(L, N, vmax, p, 500, 6), 3, CUDA)
    assert e.exchange_mode == MODE[xchg]
    e.set_checksum(False)
    e.set_state(x0, v0)
    e.advance(37)
    x, v = e.snapshot()
    assert (x == o1["x"]).all() and (v == o1["v"]).all()
    # a different state mid-run: every fifth car stopped
    x2, v2 = x.copy(), v.copy()
    v2[::5] = 0
    o2 = port.run(L, vmax, p, 6, 200, x2, v2, want_checksum=False, rng_state=o1["rng"])
    e.set_state(x2, v2)
    e.advance(200)
    x, v = e.snapshot()
    assert (x == o2["x"]).all() and (v == o2["v"]).all()
    assert (e.sumv_series()[-200:] == o2["sumv"]).all()
    e.close()


def test_distributed_checksum_single_rank(port, xchg):
    """The one-process-per-GPU ring with the trajectory checksum switched
    on: per-step piece maps all-gathered over NCCL (1-rank communicator)
    and composed on the host equal the reference's serial FNV-1a."""
    L, N, vmax, p, T = 40000, 12000, 5, 0.3, 40
    x0, v0 = nasch.fill_uniform_state(L, N, 5, 8)
    o = port.run(L, vmax, p, 3, T, x0.astype(np.uint64), v0.astype(np.uint64))
    e = nasch.Engine.distributed(mk(L, N, vmax, p, T, 3), 0, 1, nasch.nccl_unique_id())
    e.set_checksum(True)
    e.set_state(x0, v0)
    e.advance(17)
    e.advance(T)
    assert e.checksum == o["checksum"]
    x, v = e.snapshot()
    assert (x == o["x"]).all() and (v == o["v"]).all()
    e.close()


def test_distributed_whole_ring_calls_and_segment_snapshots(port, xchg, tmp_path):
    """The collective whole-ring calls of a one-process-per-GPU ring (1-rank
    communicator: the same NCCL broadcast / all-reduce / all-gather code
    paths): state gathered over ncclBroadcast, observables and series from
    the all-reduced step records, frames, set_state from the segment,
    synchronous and asynchronous segment snapshots (element k at rank
    first_rank + k), all equal to the oracle."""
    L, N, vmax, p, T = 50000, 11000, 5, 0.35, 45
    x0, v0 = nasch.fill_uniform_state(L, N, 5, 21)
    x0 = x0.astype(np.uint64)
    v0 = v0.astype(np.uint64)
    o = port.run(L, vmax, p, 8, T, x0, v0, want_checksum=False)
    e = nasch.Engine.distributed(mk(L, N, vmax, p, 200, 8, output="ascii", stride=9), 0, 1,
                                 nasch.nccl_unique_id())
    e.set_checksum(False)
    e.set_segment_state(x0, v0)  # this rank's segment = the whole ring
    e.advance(T)
    x, v = e.snapshot()
    assert (x == o["x"]).all() and (v == o["v"]).all()
    assert (e.sumv_series() == o["sumv"]).all() and (e.wrap_series() == o["wraps"]).all()
    d, m, f = e.observables()
    assert m == float(o["sumv"][-1]) / N and d == N / L
    sx, sv, first = e.segment_snapshot()
    r = (first + np.arange(N, dtype=np.uint64)) % np.uint64(N)
    assert (sx == o["x"][r]).all() and (sv == o["v"][r]).all()
    sx32, sv32, first32 = e.segment_snapshot32()  # nasch_sim_state_segment32
    assert first32 == first and (sx32 == sx).all() and (sv32 == sv).all()
    ax = np.empty(N, np.uint64)
    av = np.empty(N, np.uint64)
    first2 = e.segment_snapshot_async(ax, av)
    e.enqueue(20)  # keeps stepping while the snapshot lands
    e.snapshot_wait()
    e.synchronize()
    assert first2 == first and (ax == sx).all() and (av == sv).all()
    # frames: the single-GPU engine's, byte for byte
    a = nasch.Engine(mk(L, N, vmax, p, 200, 8, output="ascii", stride=9))
    a.set_checksum(False)
    a.set_state(x0, v0)
    a.advance(T + 20)
    assert a.frame_count == e.frame_count == (T + 20 + 8) // 9
    a.write_ascii(str(tmp_path / "a.txt"))
    e.write_ascii(str(tmp_path / "b.txt"))
    assert open(tmp_path / "a.txt").read() == open(tmp_path / "b.txt").read()
    # a rejected segment leaves the ring untouched, on every rank alike
    before = e.snapshot()
    bad = x0.copy()
    bad[5] = bad[4]
    with pytest.raises(nasch.NaschError, match="strictly increasing"):
        e.set_segment_state(bad, v0)
    with pytest.raises(nasch.NaschError, match="segment length"):
        e.set_segment_state(x0[:-1], v0[:-1])
    after = e.snapshot()
    assert (after[0] == before[0]).all() and (after[1] == before[1]).all()
    e.close()
    a.close()


def test_in_process_shards_segment_api(port):
    """Engines holding the whole ring: the segment snapshot is the rank-
    ordered state with first_rank 0 and set_state_segment is set_state."""
    L, N, vmax, p, T = 40000, 9000, 5, 0.25, 33
    x0, v0 = nasch.fill_uniform_state(L, N, 5, 3)
    x0 = x0.astype(np.uint64)
    v0 = v0.astype(np.uint64)
    o = port.run(L, vmax, p, 2, T, x0, v0, want_checksum=False)
    for G, kind in ((1, 0), (3, CUDA)):
        e = nasch.Engine(mk(L, N, vmax, p, T, 2), G, kind)
        e.set_checksum(False)
        e.set_segment_state(x0, v0)
        e.advance(T)
        sx, sv, first = e.segment_snapshot()
        assert first == 0 and (sx == o["x"]).all() and (sv == o["v"]).all()
        sx32, sv32, first32 = e.segment_snapshot32()
        assert first32 == 0 and (sx32 == sx).all() and (sv32 == sv).all()
        e.close()
