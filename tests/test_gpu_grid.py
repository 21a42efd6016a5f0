"""GPU grid-representation engine (NASCH_ENGINE_GRID_REFERENCE) against the
reference's golden values and against the agent engine, the way the
reference pins its serial grid engine (test_capi.cpp:138-155,
test_engine.cpp:224-236, acceptance.cpp:89-137)."""
import random

import numpy as np
import pytest

from paper_2309_14311_b200 import nasch

pytestmark = pytest.mark.gpu

GRID = nasch.Engine.GRID_REFERENCE
BASE = "length = 50\nncars = 10\nvmax = 3\np = 0.5\nsteps = 20\nseed = 1\n"


def test_grid_golden_checksum():
    p, _ = nasch.SimParams.parse(BASE)
    g = nasch.Engine(p, 1, GRID)
    g.run()
    assert g.checksum == 6917392272001519308
    x, v = g.snapshot()
    assert list(x) == [0, 8, 11, 17, 27, 29, 40, 43, 45, 48]
    assert list(v) == [1, 2, 2, 2, 2, 1, 3, 1, 0, 1]
    with pytest.raises(nasch.NaschError, match="serial only"):
        nasch.Engine(p, 2, GRID)


def test_grid_equals_agent_random_sweep():  # acceptance.cpp:89-137
    rd = random.Random(20260823)
    for trial in range(40):
        L = 1 + rd.randrange(300)
        N = 1 + rd.randrange(L)
        vmax = 1 + rd.randrange(7)
        p = rd.randrange(10001) / 10000.0
        T = 1 + rd.randrange(150)
        seed = rd.getrandbits(64)
        prm = nasch.SimParams(length=L, ncars=N, vmax=vmax, p=p, steps=T, seed=seed)
        a = nasch.Engine(prm, 1, nasch.Engine.AGENT)
        g = nasch.Engine(prm, 1, GRID)
        a.run()
        g.run()
        assert a.checksum == g.checksum, trial  # folds every step's state
        xa, va = a.snapshot()
        xg, vg = g.snapshot()
        assert (xa == xg).all() and (va == vg).all()
        assert (a.sumv_series() == g.sumv_series()).all()
        assert a.observables() == g.observables()


def test_grid_large_ring_vs_oracle(port):
    """Many 4096-cell blocks, injected state, crossings at the block seams."""
    L, N, vmax, p, T = 300001, 60000, 9, 0.3, 60
    x0, v0 = nasch.fill_uniform_state(L, N, vmax, 5)
    o = port.run(L, vmax, p, 9, T, x0.astype(np.uint64), v0.astype(np.uint64), want_checksum=False)
    g = nasch.Engine(nasch.SimParams(length=L, ncars=N, vmax=vmax, p=p, steps=T, seed=9), 1, GRID)
    g.set_checksum(False)
    g.set_state(x0, v0)
    g.run()
    x, v = g.snapshot()
    assert (x == o["x"]).all() and (v == o["v"]).all()
    assert (g.sumv_series() == o["sumv"]).all() and (g.wrap_series() == o["wraps"]).all()


def test_grid_device_checksum_many_chunks(port):
    """The grid engine's on-device checksum over a row of many 4096-value
    chunks (positions and velocities) equals the reference's serial fold."""
    L, N, vmax, p, T = 100003, 20011, 5, 0.35, 40
    x0, v0 = nasch.fill_uniform_state(L, N, vmax, 7)
    o = port.run(L, vmax, p, 3, T, x0.astype(np.uint64), v0.astype(np.uint64))
    g = nasch.Engine(nasch.SimParams(length=L, ncars=N, vmax=vmax, p=p, steps=T, seed=3), 1, GRID)
    g.set_state(x0, v0)
    g.advance(T)
    assert g.checksum == o["checksum"]
    x, v = g.snapshot()
    assert (x == o["x"]).all() and (v == o["v"]).all()


@pytest.mark.parametrize("L,N,vmax,p,T", [
    (8192 * 6 + 3, 9000, 9, 0.3, 50),     # a 3-cell tail block: cars jump over it into block 0
    (8192 * 5 + 100, 12000, 40, 0.2, 40),  # look > 16: the next car after a block searched past the window
    (60000, 4000, 200, 0.1, 30),           # velocities >= 128: occupancy by byte compare, not bit 7
    (8192 * 3, 24576, 5, 0.5, 20)])        # every cell occupied, L a multiple of the block
def test_grid_block_geometry_edges_vs_oracle(port, L, N, vmax, p, T):
    """grid_move3_kernel's 8192-cell blocks at their edges, against the
    oracle: spills into a non-adjacent block, the long next-car search,
    the byte-compare occupancy path and a full road."""
    x0, v0 = nasch.fill_uniform_state(L, N, min(vmax, 5), 11)
    o = port.run(L, vmax, p, 4, T, x0.astype(np.uint64), v0.astype(np.uint64), want_checksum=False)
    g = nasch.Engine(nasch.SimParams(length=L, ncars=N, vmax=vmax, p=p, steps=T, seed=4), 1, GRID)
    g.set_checksum(False)
    g.set_state(x0, v0)
    g.advance(T // 2)
    g.advance(T - T // 2)
    x, v = g.snapshot()
    assert (x == o["x"]).all() and (v == o["v"]).all()
    assert (g.sumv_series() == o["sumv"]).all() and (g.wrap_series() == o["wraps"]).all()


# --- bit-plane form (csrc/grid_bits.cuh): vmax <= 7 and L a multiple of 32 ---

@pytest.mark.parametrize("L,N,vmax,p,T", [
    (32, 5, 7, 0.3, 100),                  # one word: the carry returns into the word it left
    (64, 64, 3, 0.5, 10),                  # every cell occupied
    (96, 1, 7, 0.0, 200),                  # one car, no noise: laps of the ring through every carry
    (16384, 3000, 5, 0.13, 80),            # exactly one 512-word block
    (16384 + 32, 3500, 7, 0.4, 80),        # a one-word tail block
    (16384 * 2 + 96, 20000, 6, 0.5, 60),   # a partial tail block, jammed
    (32000, 200, 1, 0.9, 100),             # vmax = 1
    (32768 * 3, 30000, 4, 0.25, 64),       # whole blocks at 4 words per thread too
    (999968, 200000, 5, 0.25, 100)])       # ~61 blocks, C2's density
def test_grid_bit_planes_vs_oracle(port, L, N, vmax, p, T):
    """grid_bitmove_kernel against the oracle: word, warp, block and ring
    seams, a mid-run state read (planes unpacked, stepping continues from the
    planes) and the per-step series."""
    x0, v0 = nasch.fill_uniform_state(L, N, vmax, 21)
    o = port.run(L, vmax, p, 6, T, x0.astype(np.uint64), v0.astype(np.uint64))
    g = nasch.Engine(nasch.SimParams(length=L, ncars=N, vmax=vmax, p=p, steps=T, seed=6), 1, GRID)
    g.set_state(x0, v0)
    g.advance(T // 3)
    xm, vm = g.snapshot()
    assert (xm[1:] > xm[:-1]).all() and int(vm.sum()) == int(g.sumv_series()[-1])
    g.advance(T - T // 3)
    x, v = g.snapshot()
    assert (x == o["x"]).all() and (v == o["v"]).all()
    assert (g.sumv_series() == o["sumv"]).all() and (g.wrap_series() == o["wraps"]).all()
    assert g.checksum == o["checksum"]


def test_grid_bit_planes_equal_agent_and_bytes_random_sweep(monkeypatch):
    """Random rings with L a multiple of 32: the bit-plane grid, the
    byte-per-cell grid (NASCH_B200_GRID_BYTES=1) and the agent engine agree
    on every step's state (checksum), the series and the observables."""
    rd = random.Random(20261021)
    for trial in range(30):
        L = 32 * (1 + rd.randrange(40))
        N = 1 + rd.randrange(L)
        vmax = 1 + rd.randrange(7)
        p = rd.randrange(10001) / 10000.0
        T = 1 + rd.randrange(120)
        prm = nasch.SimParams(length=L, ncars=N, vmax=vmax, p=p, steps=T, seed=rd.getrandbits(64))
        a = nasch.Engine(prm, 1, nasch.Engine.AGENT)
        g = nasch.Engine(prm, 1, GRID)
        monkeypatch.setenv("NASCH_B200_GRID_BYTES", "1")
        gb = nasch.Engine(prm, 1, GRID)
        monkeypatch.delenv("NASCH_B200_GRID_BYTES")
        for e in (a, g, gb):
            e.run()
        assert a.checksum == g.checksum == gb.checksum, trial
        xa, va = a.snapshot()
        for e in (g, gb):
            xg, vg = e.snapshot()
            assert (xa == xg).all() and (va == vg).all()
            assert (a.sumv_series() == e.sumv_series()).all()
            assert a.observables() == e.observables()


@pytest.mark.parametrize("wpt", [1, 2, 4])
def test_grid_bit_planes_words_per_thread(port, monkeypatch, wpt):
    """Every instantiation of the move kernel (1, 2 or 4 words per thread;
    the engine picks by ring size, NASCH_B200_GRID_WPT forces one) on rings
    with a partial tail block for that geometry, against the oracle."""
    monkeypatch.setenv("NASCH_B200_GRID_WPT", str(wpt))
    for L, N, vmax, p, T in [(256 * wpt * 32 * 2 + 64, 9000 * wpt, 5, 0.3, 50),
                             (256 * wpt * 32, 2000 * wpt, 7, 0.6, 40), (96, 40, 2, 0.2, 30)]:
        x0, v0 = nasch.fill_uniform_state(L, N, vmax, 31)
        o = port.run(L, vmax, p, 8, T, x0.astype(np.uint64), v0.astype(np.uint64))
        g = nasch.Engine(nasch.SimParams(length=L, ncars=N, vmax=vmax, p=p, steps=T, seed=8), 1, GRID)
        g.set_state(x0, v0)
        g.run()
        x, v = g.snapshot()
        assert (x == o["x"]).all() and (v == o["v"]).all()
        assert (g.sumv_series() == o["sumv"]).all() and (g.wrap_series() == o["wraps"]).all()
        assert g.checksum == o["checksum"]


@pytest.mark.parametrize("mode", ["ascii", "pgm"])
def test_grid_bit_planes_frames_match_reference_grid_engine(tmp_path, mode):
    """Frames recorded from the bit planes (the row compacted on the device,
    steps in between on the planes) written as ascii / pgm: byte-equal to the
    files of the reference library's own grid engine (src/engine.cpp:186-196,
    src/io.cpp:140-216)."""
    import ctypes as C
    import os
    import oracle as O
    ref = C.CDLL(os.path.join(os.path.dirname(O.__file__), "_ref", "libnasch_ref.so"))
    ref.nasch_params_parse.argtypes = [C.c_char_p, C.POINTER(C.c_void_p), C.c_void_p]
    ref.nasch_sim_new_kind.argtypes = [C.c_void_p, C.c_uint, C.c_int, C.POINTER(C.c_void_p)]
    ref.nasch_sim_run.argtypes = [C.c_void_p]
    ref.nasch_sim_checksum.argtypes = [C.c_void_p]
    ref.nasch_sim_checksum.restype = C.c_uint64
    writer = getattr(ref, "nasch_sim_write_" + mode)
    writer.argtypes = [C.c_void_p, C.c_char_p]
    ref.nasch_sim_free.argtypes = [C.c_void_p]
    text = f"length=640\nncars=150\nvmax=5\np=0.35\nsteps=90\nseed=12\nstride=9\noutput={mode}"
    hp, hs = C.c_void_p(), C.c_void_p()
    assert ref.nasch_params_parse(text.encode(), C.byref(hp), None) == 0
    assert ref.nasch_sim_new_kind(hp, 1, GRID, C.byref(hs)) == 0
    assert ref.nasch_sim_run(hs) == 0
    assert writer(hs, str(tmp_path / "ref.out").encode()) == 0
    ref_checksum = ref.nasch_sim_checksum(hs)
    ref.nasch_sim_free(hs)
    p, _ = nasch.SimParams.parse(text)
    g = nasch.Engine(p, 1, GRID)
    g.run()
    assert g.frame_count == 10 and g.checksum == ref_checksum
    getattr(g, "write_" + mode)(str(tmp_path / "ours.out"))
    assert open(tmp_path / "ours.out", "rb").read() == open(tmp_path / "ref.out", "rb").read()
