"""Full-size parity for the configurations the benchmark numbers are quoted on.

Each test runs the SAME engine path the benchmark times -- default launch
geometry, temporal-blocked launches of K steps, the grid-stride tile walk
of a 2e8-car ring -- at the BASELINE.json size and compares it bit for bit
with the reference itself (oracle/_ref: the unmodified reference sources,
its OpenMP Engine on all host cores):

* C3 (L=1e9, N=2e8, p=0.13): 96 steps = three full 32-step launches, every
  step's velocity sum and crossing count, final positions and velocities.
* C5 (L=1e8, N=6e7, p=0.5, k=8 as BASELINE names it, 16 and 32): 64 steps,
  plus an asynchronous snapshot taken at step 64 while the ring keeps
  stepping.
* C4: one 64-ring slice of the fundamental-diagram sweep (every density,
  one p) for the full 5000 steps; per-ring velocity totals (the
  time-averaged flux numerators) bit-equal with the reference run ring by
  ring at one worker each (engine.cpp:101-184).
* The one-warp small-ring kernel past the device step-record ring with
  chunk lengths that are not multiples of 32.
"""
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

from paper_2309_14311_b200 import nasch

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def params(L, N, vmax, p, steps, seed):
    return nasch.SimParams(length=L, ncars=N, vmax=vmax, p=p, steps=steps, seed=seed)


@pytest.fixture
def k_env():
    old = os.environ.get("NASCH_B200_K")
    yield
    if old is None:
        os.environ.pop("NASCH_B200_K", None)
    else:
        os.environ["NASCH_B200_K"] = old


def cores(ref):
    return max(1, ref.physical_cores() or os.cpu_count() or 1)


def test_config3_full_size_three_launches_vs_reference(ref):
    """C3 exactly as bench.py runs it: 2e8 cars, two full launches of the
    default depth (K = 32 steps; enqueued one launch at a time, as the
    timed region does) and a shorter third one (8 steps), i.e. 72 steps and
    both plan hand-offs between launches (the reference's side of the check
    costs ~1.8 s per step on 16 cores)."""
    L, N, p, seed = 10**9, 2 * 10**8, 0.13, 3
    x0, v0 = nasch.fill_uniform_state(L, N, 0, seed)
    e = nasch.Engine(params(L, N, 5, p, 1000, seed))
    e.set_checksum(False)
    e.set_state(x0, v0)
    K = e.steps_per_launch
    assert K == 32
    T = 2 * K + 8
    for k in (K, K, 8):
        e.enqueue(k)
    e.synchronize()
    x, v = e.snapshot()
    sumv, wraps = e.sumv_series(), e.wrap_series()
    e.close()
    r = ref.run(L, N, 5, p, seed, T, x0=x0.astype(np.uint64), v0=v0.astype(np.uint64),
                workers=cores(ref))
    del x0, v0
    assert (sumv == r["sumv"]).all(), "per-step velocity sums differ"
    assert (wraps == r["wraps"]).all(), "per-step crossing counts differ"
    assert (x == r["x"]).all(), "positions differ"
    assert (v == r["v"]).all(), "velocities differ"


_C5 = {}


def c5_reference(ref, L, N, p, seed, T, x0, v0):
    """The reference's 64 steps of C5, run once for the three K's (it does not
    depend on K): ~30 s on 16 cores."""
    if "r" not in _C5:
        _C5["r"] = ref.run(L, N, 5, p, seed, T, x0=x0.astype(np.uint64), v0=v0.astype(np.uint64), workers=cores(ref))
    return _C5["r"]


@pytest.mark.parametrize("K", [8, 16, 32])
def test_config5_full_size_vs_reference_with_snapshot(ref, k_env, K):
    """C5 (jam-dominated, p=0.5) at k=8 (BASELINE's k), 16 and the default
    32: 64 steps,
    every step's sums/crossings, and an asynchronous snapshot at step 64
    that completes while 16 further steps run."""
    L, N, p, seed, T = 10**8, 6 * 10**7, 0.5, 5, 64
    os.environ["NASCH_B200_K"] = str(K)
    x0, v0 = nasch.fill_uniform_state(L, N, 0, seed)
    e = nasch.Engine(params(L, N, 5, p, 20000, seed))
    e.set_checksum(False)
    e.set_state(x0, v0)
    assert e.steps_per_launch == K
    e.advance(T)
    sx = np.empty(N, np.uint64)
    sv = np.empty(N, np.uint64)
    e.snapshot_async(sx, sv)
    e.enqueue(16)  # the ring keeps stepping while the snapshot lands
    e.snapshot_wait()
    e.synchronize()
    sumv, wraps = e.sumv_series()[:T], e.wrap_series()[:T]
    e.close()
    r = c5_reference(ref, L, N, p, seed, T, x0, v0)
    assert (sumv == r["sumv"]).all() and (wraps == r["wraps"]).all()
    assert (sx == r["x"]).all() and (sv == r["v"]).all()


def c4_slice(p_index=5, replica=0):
    """64 rings of BASELINE config 4: every density j, one p, one seed
    replica (the same (N, p, seed) formula as bench.py's C4 leg)."""
    ps = [0.0, 0.1, 0.2, 0.3, 0.4, 0.5, 0.6, 0.7]
    return [(5000 + (45000 * j) // 63, ps[p_index], 1 + replica * 1000 + p_index * 100 + j)
            for j in range(64)]


def test_config4_slice_full_length_vs_reference(ref):
    L, T = 10**5, 5000
    specs = c4_slice()
    ens = nasch.Ensemble([params(L, N, 5, p, T, sd) for N, p, sd in specs])
    xs, vs = [], []
    for N, _, sd in specs:
        x, v = nasch.fill_uniform_state(L, N, 0, sd)
        xs.append(x)
        vs.append(v)
    ens.set_state_all(np.concatenate(xs), np.concatenate(vs))
    ens.advance(T)
    tot, last = ens.sumv_totals(), ens.sumv_last()
    assert all(ens.steps_done(i) == T for i in range(len(specs)))
    ens.close()

    def one(i):
        N, p, sd = specs[i]
        r = ref.run(L, N, 5, p, sd, T, x0=xs[i].astype(np.uint64), v0=vs[i].astype(np.uint64),
                    workers=1, want_state=False)
        return int(r["sumv"].sum(dtype=np.uint64)), int(r["sumv"][-1])

    with ThreadPoolExecutor(cores(ref)) as pool:
        want = list(pool.map(one, range(len(specs))))
    assert [int(t) for t in tot] == [w[0] for w in want], "time-averaged flux totals differ"
    assert [int(t) for t in last] == [w[1] for w in want]


@pytest.mark.parametrize("quad", ["0", "2"])
@pytest.mark.parametrize("N", [200, 203, 509])
def test_warp_ring_past_record_ring_ragged_chunks(port, monkeypatch, N, quad):
    """The one-warp kernel (N <= 512; 200 is the EXACT instantiation) and the
    four-warp kernel (NASCH_B200_QUADRING=2: every N <= 512) over
    69,901 steps -- past the 65,536-slot device step-record ring -- in
    chunks that are not multiples of 32, against the oracle."""
    monkeypatch.setenv("NASCH_B200_QUADRING", quad)
    L, p, seed = 5 * N, 0.13, 42
    chunks = [31, 1000, 65537, 3333]
    T = sum(chunks)
    x0, v0 = nasch.fill_uniform_state(L, N, 5, 7)
    e = nasch.Engine(params(L, N, 5, p, T, seed))
    e.set_checksum(False)
    e.set_state(x0, v0)
    for c in chunks:
        e.advance(c)
    x, v = e.snapshot()
    sumv, wraps = e.sumv_series(), e.wrap_series()
    e.close()
    o = port.run(L, 5, p, seed, T, x0.astype(np.uint64), v0.astype(np.uint64), want_checksum=False)
    assert len(sumv) == T
    assert (sumv == o["sumv"]).all() and (wraps == o["wraps"]).all()
    assert (x == o["x"]).all() and (v == o["v"]).all()


@pytest.mark.parametrize("N,vmax", [(65, 3), (128, 5), (129, 5), (256, 7), (257, 2), (384, 5), (511, 5), (512, 300)])
def test_quad_ring_every_instantiation_vs_oracle(port, monkeypatch, N, vmax):
    """ring_quad_kernel (four warps, 1 / 2 / 4 cars per thread, exact and
    ragged, u8 and u32 velocities) with the checksum on (row dumps) and a
    chunked advance, against the oracle."""
    monkeypatch.setenv("NASCH_B200_QUADRING", "2")
    L, p, seed, T = 4 * N + 3, 0.3, 9, 700
    x0, v0 = nasch.fill_uniform_state(L, N, min(vmax, 5), 13)
    e = nasch.Engine(params(L, N, vmax, p, T, seed))
    e.set_state(x0, v0)
    e.advance(333)
    e.advance(T - 333)
    x, v = e.snapshot()
    o = port.run(L, vmax, p, seed, T, x0.astype(np.uint64), v0.astype(np.uint64))
    assert (x == o["x"]).all() and (v == o["v"]).all()
    assert (e.sumv_series() == o["sumv"]).all() and (e.wrap_series() == o["wraps"]).all()
    assert e.checksum == o["checksum"]
    e.close()


@pytest.mark.parametrize("dr_min", ["512", "4096"])
@pytest.mark.parametrize("N", [513, 600, 2000, 4096])
def test_rings_of_513_to_4096_cars_both_engines_vs_oracle(port, monkeypatch, N, dr_min):
    """513..4096 cars: the distributed-resident kernel (default from 513 cars:
    0.44 us per step against 0.9-1.3 on one CTA) and the one-CTA shared-memory
    kernel (NASCH_B200_DR_MIN=4096; still the path of u32-velocity rings),
    checksum on, chunked advance, against the oracle."""
    monkeypatch.setenv("NASCH_B200_DR_MIN", dr_min)
    L, p, seed, T = 4 * N + 1, 0.25, 17, 300
    x0, v0 = nasch.fill_uniform_state(L, N, 5, 19)
    e = nasch.Engine(params(L, N, 5, p, T, seed))
    e.set_state(x0, v0)
    e.advance(101)
    e.advance(T - 101)
    x, v = e.snapshot()
    o = port.run(L, 5, p, seed, T, x0.astype(np.uint64), v0.astype(np.uint64))
    assert (x == o["x"]).all() and (v == o["v"]).all()
    assert (e.sumv_series() == o["sumv"]).all() and (e.wrap_series() == o["wraps"]).all()
    assert e.checksum == o["checksum"]
    e.close()


@pytest.mark.parametrize("L,N,vmax,p,T", [
    (5 * 20000, 20000, 5, 0.3, 70),       # forced onto few, mostly empty 32-car threads
    (3 * 640000, 640000, 5, 0.25, 64),    # 20 cars per thread (564k..715k cars), density 1/3
    (2 * 800000, 800000, 7, 0.1, 48),     # 24 cars per thread (..865k cars)
    (1150000 + 7, 1150000, 3, 0.5, 40)])  # near its capacity, an almost full road
def test_dr_32_cars_per_thread_vs_oracle(port, monkeypatch, L, N, vmax, p, T):
    """ring_dr_kernel<u8,256,20|24|32,QDRAW> (draws from one per-thread base
    times 2 a^c; rings of 0.56M..1.17M cars, or NASCH_B200_DR_GEOM=3..5) against the
    oracle: state, both series, checksum, a chunked advance across launches."""
    if N < 564000:
        monkeypatch.setenv("NASCH_B200_DR_GEOM", "5")
    x0, v0 = nasch.fill_uniform_state(L, N, vmax, 23)
    e = nasch.Engine(params(L, N, vmax, p, T, 29))
    assert e.steps_per_launch > 32  # the distributed-resident engine
    e.set_state(x0, v0)
    e.advance(33)
    e.advance(T - 33)
    x, v = e.snapshot()
    o = port.run(L, vmax, p, 29, T, x0.astype(np.uint64), v0.astype(np.uint64))
    assert (x == o["x"]).all() and (v == o["v"]).all()
    assert (e.sumv_series() == o["sumv"]).all() and (e.wrap_series() == o["wraps"]).all()
    assert e.checksum == o["checksum"]
    e.close()
