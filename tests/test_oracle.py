"""Pins the CPU oracle (oracle/nasch_oracle.c) before it is trusted.

Golden vectors are the reference's own known-answer tests (their doctest
suites cannot build here: vendor/doctest.h is absent), restated with the
file:line they come from, plus cross-checks against oracle/_ref -- the
reference sources compiled unmodified.
"""
import random

import numpy as np
import pytest

import oracle as O

M = O.M


# ---- PRNG: tests/test_lcg.cpp ---------------------------------------------

def test_first_draws(port):  # test_lcg.cpp:13-18
    assert port.next(port.seeded(1))[0] == 48271
    assert port.next(port.seeded(2))[0] == 96542


def test_seeding_escape(port):  # test_lcg.cpp:20-26
    assert port.seeded(1) == 1
    assert port.seeded(0) == 1
    assert port.seeded(2147483647) == 1
    assert port.seeded(2147483647 + 5) == 5
    assert port.seeded(7) == 7


def test_minstd_rand_sequence(port):  # test_lcg.cpp:28-34 (std::minstd_rand)
    s = port.seeded(20260823)
    py = 20260823 % M
    for _ in range(1000):
        r, s = port.next(s)
        py = (48271 * py) % M
        assert r == py


def test_ten_thousandth_draw(port):  # test_lcg.cpp:36-41
    s = port.seeded(1)
    for _ in range(10000):
        r, s = port.next(s)
    assert r == 399268537


JUMP_ROWS = [  # test_lcg.cpp:51-62
    (1, 2, 182605794), (1, 7, 1105902161), (1, 100, 1358404307),
    (1, 12345, 1941600346), (1, 1000000, 1263606197), (42, 1, 2027382),
    (42, 2, 1226992407), (42, 7, 1350734175), (42, 100, 1218406072),
    (42, 12345, 2090319593), (42, 1000000, 1531852746),
    (1073741824, 1, 1073765959), (1073741824, 2, 91302897),
    (1073741824, 7, 1626692904), (1073741824, 100, 1752943977),
    (1073741824, 12345, 970800173), (1073741824, 1000000, 1705544922),
]


@pytest.mark.parametrize("seed,span,state", JUMP_ROWS)
def test_frozen_jumps(port, seed, span, state):
    assert port.jump(port.seeded(seed), span) == state
    # the counter-based form the GPU uses: s0 * a^k mod m
    assert port.seeded(seed) * pow(48271, span, M) % M == state


def test_jump_identities(port):  # test_lcg.cpp:72-98, 100-121
    assert port.jump(port.seeded(123), 0) == port.seeded(123)
    assert port.jump(port.seeded(99), 1) == port.next(port.seeded(99))[1]
    for k1 in (0, 1, 3, 17, 1000):
        for k2 in (0, 2, 5, 999):
            assert port.jump(port.jump(port.seeded(7), k1), k2) == port.jump(port.seeded(7), k1 + k2)
    assert port.jump_coefficients(0) == (1, 0)
    assert port.jump_coefficients(1) == (48271, 0)
    assert port.jump_coefficients(1000000) == (1263606197, 0)


def test_uniform01(port):  # test_lcg.cpp:135-156
    u, _ = port.uniform01(port.seeded(1))
    assert u == 48271.0 / 2147483647.0
    s = port.seeded(1)
    total = 0.0
    for _ in range(200000):
        u, s = port.uniform01(s)
        total += u
    # the reference pins the 1e6-draw mean at 0.4997635306662361; check a
    # prefix for speed and the full value through oracle/_ref below
    assert 0.49 < total / 200000 < 0.51


# ---- model: tests/test_model.cpp -------------------------------------------

def test_init_state(port):  # test_model.cpp:71-86
    x, v = port.init_state(1000, 200)
    assert list(x) == [5 * i for i in range(200)] and not v.any()
    x, _ = port.init_state(10, 3)
    assert list(x) == [0, 3, 6]


def test_gap_ahead(port):  # test_model.cpp:88-108
    assert [port.gap_ahead([0, 2, 7], 10, i) for i in range(3)] == [1, 4, 2]
    assert port.gap_ahead([11], 25, 0) == 24
    assert [port.gap_ahead([0, 1, 2, 3], 4, i) for i in range(4)] == [0, 0, 0, 0]


def test_lone_car_free_acceleration(port):  # test_model.cpp:110-132
    x, v = port.init_state(100, 1)
    s = port.seeded(1)
    for t, (wx, wv) in enumerate(zip([1, 3, 6, 10, 15], [1, 2, 3, 4, 5])):
        _, s = port.step(x, v, 100, 5, 0.0, s)
        assert (x[0], v[0]) == (wx, wv)
    for _ in range(50):
        _, s = port.step(x, v, 100, 5, 0.0, s)
        assert v[0] == 5


def test_p1_never_moves(port):  # test_model.cpp:134-149
    x, v = port.init_state(100, 1)
    s = port.seeded(7)
    for _ in range(100):
        _, s = port.step(x, v, 100, 5, 1.0, s)
        assert x[0] == 0 and v[0] == 0


@pytest.mark.parametrize("p", [0.0, 0.5, 1.0])
def test_full_ring_fixed_point(port, p):  # test_model.cpp:151-170
    x, v = port.init_state(12, 12)
    x0 = x.copy()
    s = port.seeded(3)
    for _ in range(100):
        _, s = port.step(x, v, 12, 5, p, s)
        assert (x == x0).all() and not v.any()


def test_brake_clamp(port):  # test_model.cpp:172-188
    x = np.array([0, 2], np.uint64)
    v = np.array([4, 0], np.uint64)
    port.step(x, v, 10, 5, 0.0, port.seeded(1))
    assert list(x) == [1, 3] and list(v) == [1, 1]


def test_draws_per_step(port):  # test_model.cpp:190-210
    x, v = port.init_state(50, 10)
    s = port.seeded(1)
    for _ in range(20):
        want = port.jump(s, 10)
        _, s = port.step(x, v, 50, 3, 0.5, s)
        assert s == want


def test_frozen_twenty_step_endpoint(port):  # test_model.cpp:233-243
    x, v = port.init_state(50, 10)
    r = port.run(50, 3, 0.5, 1, 20, x, v)
    assert list(r["x"]) == [0, 8, 11, 17, 27, 29, 40, 43, 45, 48]
    assert list(r["v"]) == [1, 2, 2, 2, 2, 1, 3, 1, 0, 1]


def test_grid_tracks_agent(port):  # test_model.cpp:261-274
    x, v = port.init_state(50, 10)
    cells = np.full(50, -1, np.int64)
    cells[x.astype(np.int64)] = v.astype(np.int64)
    sa = sg = port.seeded(1)
    for _ in range(100):
        _, sa = port.step(x, v, 50, 3, 0.5, sa)
        sg = port.step_grid(cells, 50, 3, 0.5, sg)
        want = np.full(50, -1, np.int64)
        want[x.astype(np.int64)] = v.astype(np.int64)
        assert (cells == want).all() and sa == sg


# ---- checksum: tests/test_engine.cpp ---------------------------------------

def test_fnv_constants(port):  # test_engine.cpp:85-115
    assert port.fnv_value(O.FNV_BASIS, 0) == 12161962213042174405
    assert port.hash_row(O.FNV_BASIS, [0], [0]) == 9808874869469701221


def test_frozen_checksum(port):  # test_engine.cpp:111-114, test_capi.cpp:478-479
    x, v = port.init_state(50, 10)
    r = port.run(50, 3, 0.5, 1, 20, x, v)
    assert r["checksum"] == 6917392272001519308
    assert r["rng"] == port.jump(port.seeded(1), 200)  # draws = 200


# ---- oracle vs the reference itself (oracle/_ref) --------------------------

def test_ref_build_matches_golden(ref):
    r = ref.run(50, 10, 3, 0.5, 1, 20)
    assert r["checksum"] == 6917392272001519308
    assert list(r["x"]) == [0, 8, 11, 17, 27, 29, 40, 43, 45, 48]
    # W-invariance of the reference itself (test_engine.cpp:136-152)
    a = ref.run(137, 61, 5, 0.3, 2026, 150, workers=1)
    for w in (2, 3, 5, 8, 13, 61, 100):
        b = ref.run(137, 61, 5, 0.3, 2026, 150, workers=w)
        assert b["checksum"] == a["checksum"]


def test_oracle_equals_reference_random_sweep(port, ref):
    """acceptance.cpp:89-137 style sweep, oracle vs reference, step by step
    (per-step velocity sums) and at the end (state + checksum)."""
    rd = random.Random(20260823)
    for _ in range(60):
        L = 1 + rd.randrange(300)
        N = 1 + rd.randrange(L)
        vmax = 1 + rd.randrange(7)
        p = rd.randrange(10001) / 10000.0
        T = 1 + rd.randrange(200)
        seed = rd.getrandbits(64)
        x, v = port.init_state(L, N)
        a = port.run(L, vmax, p, seed, T, x, v)
        b = ref.run(L, N, vmax, p, seed, T, workers=1 + rd.randrange(4))
        assert (a["x"] == b["x"]).all() and (a["v"] == b["v"]).all()
        assert (a["sumv"] == b["sumv"]).all()
        assert a["checksum"] == b["checksum"]


def test_oracle_equals_reference_injected_state(port, ref):
    """Injected (non-equally-spaced) initial states -- the BASELINE inits."""
    rd = np.random.default_rng(5)
    for trial in range(20):
        L = int(rd.integers(5, 5000))
        N = int(rd.integers(1, L + 1))
        vmax = int(rd.integers(1, 9))
        x0 = np.sort(rd.choice(L, N, replace=False)).astype(np.uint64)
        v0 = rd.integers(0, vmax + 1, N).astype(np.uint64)
        p = float(rd.random())
        a = port.run(L, vmax, p, trial, 50, x0, v0)
        b = ref.run(L, N, vmax, p, trial, 50, x0=x0, v0=v0, workers=3)
        assert (a["x"] == b["x"]).all() and (a["v"] == b["v"]).all()
        assert (a["sumv"] == b["sumv"]).all() and a["checksum"] == b["checksum"]
        assert (a["wraps"] == b["wraps"]).all()  # the reference's own wrap_counts_


def test_reference_uniform_mean_pin(ref, port):
    """test_lcg.cpp:151-156: mean of 1e6 uniforms from seed 1, computed by
    the oracle port in one pass."""
    import ctypes as C
    s = C.c_uint64(port.seeded(1))
    total = 0.0
    f = port.lib.or_uniform01
    for _ in range(1000000):
        total += f(C.byref(s))
    assert abs(total / 1e6 - 0.4997635306662361) <= 1e-12 * 0.4997635306662361


@pytest.mark.parametrize("L,N,vmax_init,seed", [
    (1000, 200, 0, 42), (10**6, 2 * 10**5, 5, 7), (50, 50, 3, 1), (50, 49, 3, 2),
    (97, 1, 5, 3), (10**5, 5000, 0, 11), (3 * 10**7, 100, 5, 3)])
def test_input_generator_matches_library(port, L, N, vmax_init, seed):
    """The oracle's restatement of the BASELINE input generator (used by the
    reference arm, which must not load the product library) equals the
    library's nasch_fill_uniform_state value for value."""
    from paper_2309_14311_b200 import nasch
    a = port.fill_uniform_state(L, N, vmax_init, seed)
    b = nasch.fill_uniform_state(L, N, vmax_init, seed)
    assert (a[0] == b[0]).all() and (a[1] == b[1]).all()
    assert len(a[0]) == N and (np.diff(a[0].astype(np.int64)) > 0).all() and int(a[0][-1]) < L
    assert int(a[1].max()) <= vmax_init
