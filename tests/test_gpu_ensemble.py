"""GPU parity of the ensemble engine (BASELINE config 4 shape) against the
oracle: every ring is the reference's single-ring model with its own
parameters and minstd stream (src/model.cpp:42-75, src/lcg.cpp:11-16)."""
import numpy as np
import pytest

from paper_2309_14311_b200 import nasch

pytestmark = pytest.mark.gpu


def mk(L, N, vmax, p, steps, seed):
    return nasch.SimParams(length=L, ncars=N, vmax=vmax, p=p, steps=steps, seed=seed)


def oracle_ring(port, L, N, vmax, p, seed, T, x0=None, v0=None):
    if x0 is None:
        x0, v0 = port.init_state(L, N)
    return port.run(L, vmax, p, seed, T, np.asarray(x0, np.uint64), np.asarray(v0, np.uint64),
                    want_checksum=False)


def test_ensemble_matches_oracle_per_ring(port):
    rng = np.random.default_rng(3)
    specs = []
    for i in range(40):
        L = int(rng.integers(20, 60000))
        N = int(rng.integers(1, min(L, 50000) + 1))
        vmax = int(rng.integers(1, 12))
        p = float(rng.choice([0.0, 0.1, 0.13, 0.3, 0.5, 0.7, 1.0]))
        specs.append((L, N, vmax, p, 120, int(rng.integers(0, 2**40))))
    ens = nasch.Ensemble([mk(*s) for s in specs])
    ens.advance(45)
    ens.advance(1000)  # clamps at 120
    tot = ens.sumv_totals()
    last = ens.sumv_last()
    for r, (L, N, vmax, p, T, seed) in enumerate(specs):
        o = oracle_ring(port, L, N, vmax, p, seed, T)
        x, v = ens.snapshot(r)
        assert ens.steps_done(r) == T
        assert (x == o["x"]).all() and (v == o["v"]).all(), r
        assert int(tot[r]) == int(o["sumv"].sum()), r
        assert int(last[r]) == int(o["sumv"][-1]), r


@pytest.fixture
def tiled_env():
    import os
    old = os.environ.get("NASCH_B200_ENS_TILED")
    yield os.environ
    if old is None:
        os.environ.pop("NASCH_B200_ENS_TILED", None)
    else:
        os.environ["NASCH_B200_ENS_TILED"] = old


@pytest.mark.parametrize("tiled", ["1", "0"])
def test_ensemble_per_step_series_and_injected_state(port, tiled_env, tiled):
    """Per-step velocity sums and injected states, through the warp-tile
    ensemble step (ensemble_tb.cuh) and the shared-memory one."""
    tiled_env["NASCH_B200_ENS_TILED"] = tiled
    specs = [(100000, 5000, 5, 0.13, 60, 11), (100000, 50000, 5, 0.7, 60, 12),
             (100000, 27500, 5, 0.0, 60, 13), (1000, 1000, 5, 0.4, 60, 14)]
    ens = nasch.Ensemble([mk(*s) for s in specs])
    inits = []
    for r, (L, N, vmax, p, T, seed) in enumerate(specs):
        x0, v0 = nasch.fill_uniform_state(L, N, 0, 100 + r)
        ens.set_state(r, x0, v0)
        inits.append((x0, v0))
    orc = [oracle_ring(port, L, N, vmax, p, seed, T, *inits[r])
           for r, (L, N, vmax, p, T, seed) in enumerate(specs)]
    for t in range(60):
        ens.advance(1)
        last = ens.sumv_last()
        for r in range(len(specs)):
            assert int(last[r]) == int(orc[r]["sumv"][t]), (r, t)
    for r in range(len(specs)):
        x, v = ens.snapshot(r)
        assert (x == orc[r]["x"]).all() and (v == orc[r]["v"]).all()


def test_ensemble_overflow_ring_and_order_invariance(port):
    """A ring too large for shared memory runs on its own engine; results do
    not depend on which rings share the launch or in which order."""
    specs = [(300000, 90000, 5, 0.2, 40, 5), (5000, 2000, 5, 0.2, 40, 6),
             (20000, 15000, 200, 0.25, 40, 7)]
    a = nasch.Ensemble([mk(*s) for s in specs])
    a.advance(40)
    b = nasch.Ensemble([mk(*s) for s in reversed(specs)])
    b.advance(17)
    b.advance(23)
    ta, tb = a.sumv_totals(), b.sumv_totals()[::-1]
    assert (ta == tb).all()
    for r, (L, N, vmax, p, T, seed) in enumerate(specs):
        o = oracle_ring(port, L, N, vmax, p, seed, T)
        x, v = a.snapshot(r)
        assert (x == o["x"]).all() and (v == o["v"]).all()
        assert int(ta[r]) == int(o["sumv"].sum())


def test_ensemble_equals_single_ring_engine():
    L, N = 100000, 35000
    x0, v0 = nasch.fill_uniform_state(L, N, 0, 9)
    e = nasch.Engine(mk(L, N, 5, 0.3, 500, 77))
    e.set_checksum(False)
    e.set_state(x0, v0)
    e.run()
    ens = nasch.Ensemble([mk(L, N, 5, 0.3, 500, 77)])
    ens.set_state(0, x0, v0)
    ens.advance(500)
    xe, ve = e.snapshot()
    xs, vs = ens.snapshot(0)
    assert (xe == xs).all() and (ve == vs).all()
    assert int(ens.sumv_totals()[0]) == int(e.sumv_series().sum())


def test_tiled_ensemble_random_rings(port, tiled_env):
    """The warp-tile ensemble on rings of every awkward size: shorter than
    one warp tile (the tile wraps several times), 496..512 cars, N not a
    multiple of 16, dense jams, vmax up to 31, p in {0, 1}, and rings with
    fewer configured steps than the others (they stop; the rest go on)."""
    tiled_env["NASCH_B200_ENS_TILED"] = "1"
    rng = np.random.default_rng(11)
    specs = []
    for i in range(48):
        vmax = int(rng.choice([1, 2, 5, 9, 31]))
        L = int(rng.integers(16 * vmax + 1, 120000))
        nmin = 16 * (vmax + 1)
        if nmin > L:
            continue
        N = int(rng.choice([nmin, 300, 496, 497, 511, 512, 1000, 4095, int(rng.integers(nmin, L + 1))]))
        N = max(nmin, min(N, L))
        p = float(rng.choice([0.0, 0.13, 0.5, 1.0]))
        T = int(rng.choice([37, 80]))
        specs.append((L, N, vmax, p, T, int(rng.integers(0, 2**40))))
    ens = nasch.Ensemble([mk(*s) for s in specs])
    ens.advance(21)
    ens.advance(1000)  # each ring clamps at its own T
    tot = ens.sumv_totals()
    last = ens.sumv_last()
    for r, (L, N, vmax, p, T, seed) in enumerate(specs):
        o = oracle_ring(port, L, N, vmax, p, seed, T)
        x, v = ens.snapshot(r)
        assert ens.steps_done(r) == T, r
        assert (x == o["x"]).all() and (v == o["v"]).all(), (r, specs[r])
        assert int(tot[r]) == int(o["sumv"].sum()), r
        assert int(last[r]) == int(o["sumv"][-1]), r


@pytest.mark.parametrize("pinned", [False, True])
def test_ensemble_set_state_all32_pinned_and_rejects(port, pinned):
    """set_state_all32 (every ring in one call): from page-locked arrays the
    positions are scattered into the tiled layout and checked on the device
    (ens_load_kernel / ens_commit_kernel), from pageable ones on the host;
    both give the oracle's trajectories, the same first-violation message
    (earliest car over all rings, rule order within a car), and a rejected
    state leaves every ring as it was."""
    import torch

    def host(a):
        if not pinned:
            return np.array(a, np.uint32)
        t = torch.empty(len(a), dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
        t[:] = a
        return t

    specs = [(30000 + 1000 * i, 5000 + 1000 * i, 5, 0.1 * (i % 6), 60, 100 + i) for i in range(24)]
    xs, vs = zip(*[nasch.fill_uniform_state(L, N, 5, sd) for (L, N, _, _, _, sd) in specs])
    xc, vc = np.concatenate(xs), np.concatenate(vs)
    ens = nasch.Ensemble([mk(*s) for s in specs])
    ens.set_state_all(host(xc), host(vc))
    ens.advance(13)
    before = [ens.snapshot(r) for r in range(len(specs))]
    starts = np.cumsum([0] + [s[1] for s in specs])
    cases = [(int(starts[5]) + 3, "x", "position out of range"), (int(starts[11]) + 7, "x2", "strictly increasing"),
             (int(starts[2]) + 9, "v", "above vmax"), (int(starts[20]) + 1, "v", "above vmax")]
    for pos, what, msg in cases:
        x, v = host(xc), host(vc)
        if what == "x":
            x[pos] = 10**6
        elif what == "x2":
            x[pos] = x[pos - 1]
        else:
            v[pos] = 6
        with pytest.raises(nasch.NaschError, match=msg):
            ens.set_state_all(x, v)
        for r in range(len(specs)):
            bx, bv = ens.snapshot(r)
            assert (bx == before[r][0]).all() and (bv == before[r][1]).all(), (msg, r)
    # the earlier car wins across rings and checks (a velocity in ring 3 before a position in ring 9)
    x, v = host(xc), host(vc)
    v[int(starts[3]) + 2] = 7
    x[int(starts[9]) + 1] = 10**6
    with pytest.raises(nasch.NaschError, match="above vmax"):
        ens.set_state_all(x, v)
    ens.set_state_all(host(xc), host(vc))
    ens.advance(60)
    for r, (L, N, vmax, p, T, sd) in enumerate(specs):
        # set_state keeps the step count: the stream continues at draw 13 N
        o = port.run(L, vmax, p, sd, T - 13, np.asarray(xs[r], np.uint64), np.asarray(vs[r], np.uint64),
                     want_checksum=False, rng_state=port.jump(port.seeded(sd), 13 * N))
        x, v = ens.snapshot(r)
        assert ens.steps_done(r) == T
        assert (x == o["x"]).all() and (v == o["v"]).all(), r
