"""The committed golden vectors (tests/golden/reference_vectors.json, written
by tests/golden/make_golden.py from the reference itself -- oracle/_ref, the
unmodified sources) against: the C restatement of the algorithm (CPU, pins the
oracle where /root/reference is absent), the reference library when it is
present, and the CUDA engines through the C ABI (GPU)."""
import hashlib
import json
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
with open(os.path.join(HERE, "golden", "reference_vectors.json")) as f:
    GOLDEN = json.load(f)["records"]
IDS = [r["name"] for r in GOLDEN]


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, np.dtype("<u8")).tobytes()).hexdigest()


def initial_state(port, r):
    """(x0, v0) as u64 arrays: the recorded generator call, or the reference's
    init_state (src/model.cpp:30-40) through the oracle's restatement."""
    st = r["state"]
    if st is None:
        x0, v0 = port.init_state(r["L"], r["N"])
    else:
        x0, v0 = port.fill_uniform_state(r["L"], r["N"], st["vmax_init"], st["seed"])
    x0, v0 = np.asarray(x0, np.uint64), np.asarray(v0, np.uint64)
    if st is not None:
        assert sha(x0) == st["x0_sha256"] and sha(v0) == st["v0_sha256"]
        if "x0" in st:
            assert list(x0) == st["x0"] and list(v0) == st["v0"]
    return x0, v0


def check(r, x, v, sumv, wraps, checksum):
    assert checksum == r["checksum"]
    assert sha(x) == r["x_sha256"] and sha(v) == r["v_sha256"]
    if "x" in r:
        assert [int(a) for a in x] == r["x"] and [int(a) for a in v] == r["v"]
    assert [int(s) for s in sumv] == r["sumv"]
    assert [int(w) for w in wraps] == r["wraps"]


def test_frozen_reference_values_are_in_the_file():
    """The reference's own known answers (tests/test_capi.cpp:105-119)."""
    r = GOLDEN[0]
    assert r["checksum"] == 6917392272001519308
    assert r["x"] == [0, 8, 11, 17, 27, 29, 40, 43, 45, 48]
    assert r["v"] == [1, 2, 2, 2, 2, 1, 3, 1, 0, 1]


@pytest.mark.parametrize("r", GOLDEN, ids=IDS)
def test_oracle_port_reproduces_golden(port, r):
    x0, v0 = initial_state(port, r)
    o = port.run(r["L"], r["vmax"], r["p"], r["seed"], r["steps"], x0, v0)
    check(r, o["x"], o["v"], o["sumv"], o["wraps"], o["checksum"])


def test_golden_file_matches_the_reference_when_present(port):
    """Where oracle/_ref exists (the build container, and the GPU box through
    the snapshot), the file is what the reference returns now."""
    import oracle as O
    if not os.path.exists(O.REF_SO):
        pytest.skip("oracle/_ref not built")
    ref = O.Ref()
    for r in GOLDEN:
        if r["N"] > 6000:
            continue
        x0 = v0 = None
        if r["state"] is not None:
            x0, v0 = initial_state(port, r)
        o = ref.run(r["L"], r["N"], r["vmax"], r["p"], r["seed"], r["steps"], workers=min(2, r["N"]), x0=x0, v0=v0)
        check(r, o["x"], o["v"], o["sumv"], o["wraps"], o["checksum"])


@pytest.mark.gpu
@pytest.mark.parametrize("r", GOLDEN, ids=IDS)
def test_cuda_agent_engine_reproduces_golden(port, r):
    from paper_2309_14311_b200 import nasch
    e = nasch.Engine(nasch.SimParams(length=r["L"], ncars=r["N"], vmax=r["vmax"], p=r["p"], steps=r["steps"],
                                     seed=r["seed"]))
    if r["state"] is not None:
        x0, v0 = initial_state(port, r)
        e.set_state(x0, v0)
    e.run()
    x, v = e.snapshot()
    check(r, x, v, e.sumv_series(), e.wrap_series(), e.checksum)
    e.close()


@pytest.mark.gpu
@pytest.mark.parametrize("r", [g for g in GOLDEN if g["N"] <= 6000 and min(g["vmax"], g["L"] - 1) <= 254],
                         ids=[g["name"] for g in GOLDEN if g["N"] <= 6000 and min(g["vmax"], g["L"] - 1) <= 254])
def test_cuda_grid_engine_reproduces_golden(port, r):
    from paper_2309_14311_b200 import nasch
    e = nasch.Engine(nasch.SimParams(length=r["L"], ncars=r["N"], vmax=r["vmax"], p=r["p"], steps=r["steps"],
                                     seed=r["seed"]), 1, nasch.Engine.GRID_REFERENCE)
    if r["state"] is not None:
        x0, v0 = initial_state(port, r)
        e.set_state(x0, v0)
    e.run()
    x, v = e.snapshot()
    check(r, x, v, e.sumv_series(), e.wrap_series(), e.checksum)
    e.close()
