"""CPU-side checks of libnasch_b200.so: it loads, exports every symbol
include/nasch/nasch.h declares, and its host plumbing (parameter sets,
parsing, validation, error folding, input generator, draw threshold)
behaves like the reference's (tests/test_capi.cpp, tests/test_io.cpp),
checked directly against oracle/_ref's own C ABI where the reference
defines the behaviour.  No compute call needs a GPU here.
"""
import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_2309_14311_b200 import capi, nasch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "nasch", "nasch.h")
REF_HEADER = "/root/reference/proj/include/nasch/nasch.h"


def _declared(path):
    text = open(path).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return set(re.findall(r"\b(nasch_\w+)\s*\(", text))


def test_header_symbols_exported(lib):
    names = _declared(HEADER)
    assert len(names) >= 36 + 12
    for name in names:
        assert hasattr(lib, name), name
        assert name in capi.SIGNATURES, name


def test_reference_abi_is_covered():
    ours = _declared(HEADER)
    ref = _declared(REF_HEADER) if os.path.exists(REF_HEADER) else set(capi.REFERENCE_SYMBOLS)
    assert len(ref) == 36
    assert ref <= ours
    assert set(capi.REFERENCE_SYMBOLS) == ref


def test_version(lib):
    assert b"sm_100a" in lib.nasch_b200_version()


# ---- test_capi.cpp:25-42, 44-62 -------------------------------------------

def test_defaults_and_roundtrip():
    p = nasch.SimParams()
    assert (p.length, p.ncars, p.vmax, p.steps, p.seed, p.stride) == (0, 0, 5, 0, 0, 1)
    assert p.p == pytest.approx(0.13) and p.output == "none"
    with pytest.raises(nasch.NaschError):
        p.validate()
    p.length, p.ncars, p.vmax, p.p, p.steps, p.seed, p.output, p.stride = 200, 40, 4, 0.25, 99, 321, "pgm", 5
    assert (p.length, p.ncars, p.vmax, p.p, p.steps, p.seed, p.output, p.stride) == \
        (200, 40, 4, 0.25, 99, 321, "pgm", 5)
    p.validate()


def test_parse_threads_and_errors(lib):
    p, threads = nasch.SimParams.parse("length=100\nncars=10\nsteps=5\nseed=2\nthreads=6\n")
    assert threads == 6 and p.length == 100
    h = C.c_void_p(1234)
    assert lib.nasch_params_parse(b"length=100\nwheels=3\n", C.byref(h), None) == capi.NASCH_ERR_PARSE
    assert b"wheels" in lib.nasch_last_error()
    assert not h.value


def test_missing_file_is_io_error(lib):
    h = C.c_void_p()
    assert lib.nasch_params_load(b"no/such/file.params", C.byref(h), None) == capi.NASCH_ERR_IO
    assert len(lib.nasch_last_error()) > 0


def test_null_arguments(lib):  # test_capi.cpp:92-103
    assert lib.nasch_params_new(None) == capi.NASCH_ERR_INVALID
    assert lib.nasch_params_parse(None, None, None) == capi.NASCH_ERR_INVALID
    assert lib.nasch_params_validate(None) == capi.NASCH_ERR_INVALID
    assert lib.nasch_sim_new(None, 1, None) == capi.NASCH_ERR_INVALID
    assert lib.nasch_sim_advance(None, 1) == capi.NASCH_ERR_INVALID
    assert lib.nasch_sim_run(None) == capi.NASCH_ERR_INVALID
    assert lib.nasch_sim_steps_done(None) == 0
    assert lib.nasch_sim_checksum(None) == 0
    lib.nasch_params_free(None)
    lib.nasch_sim_free(None)
    assert lib.nasch_sim_set_state(None, None, None, 0) == capi.NASCH_ERR_INVALID
    assert lib.nasch_sim_cuda_stream(None) is None
    # round-2 extensions: NULL handles and arrays are refused, never followed
    assert lib.nasch_sim_state_segment(None, None, None, 0, None) == capi.NASCH_ERR_INVALID
    assert lib.nasch_sim_state_segment_async(None, None, None, 0, None) == capi.NASCH_ERR_INVALID
    assert lib.nasch_sim_set_state_segment(None, None, None, 0) == capi.NASCH_ERR_INVALID
    assert lib.nasch_sim_state32(None, None, None, 0) == capi.NASCH_ERR_INVALID
    assert lib.nasch_sim_state_segment32(None, None, None, 0, None) == capi.NASCH_ERR_INVALID
    assert lib.nasch_ensemble_set_state_all32(None, None, None, 0) == capi.NASCH_ERR_INVALID
    assert lib.nasch_sim_state_wait(None) == capi.NASCH_ERR_INVALID
    assert lib.nasch_sim_exchange_mode(None) == 0
    assert b"null" in lib.nasch_last_error()


def test_invalid_params_cannot_start(lib):  # test_capi.cpp:159-166
    p = nasch.SimParams()
    h = C.c_void_p(99)
    assert lib.nasch_sim_new(p._h, 1, C.byref(h)) == capi.NASCH_ERR_INVALID
    assert not h.value
    p2, _ = nasch.SimParams.parse("length=50\nncars=10\nsteps=20\nseed=1\n")
    assert lib.nasch_sim_new(p2._h, 0, C.byref(h)) == capi.NASCH_ERR_INVALID
    assert lib.nasch_sim_new_kind(p2._h, 2, capi.NASCH_ENGINE_GRID_REFERENCE, C.byref(h)) == \
        capi.NASCH_ERR_INVALID
    assert lib.nasch_sim_new_kind(p2._h, 1, 7, C.byref(h)) == capi.NASCH_ERR_INVALID
    assert b"unknown engine kind" in lib.nasch_last_error()


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_has_gpu(), reason="checks the no-GPU failure mode")
def test_no_gpu_fails_loudly(lib):
    p, _ = nasch.SimParams.parse("length=50\nncars=10\nsteps=20\nseed=1\n")
    with pytest.raises(nasch.NaschError, match="CUDA"):
        nasch.Engine(p)


# ---- parse / validation messages vs the reference's own library ------------

BAD_TEXTS = [  # tests/test_io.cpp:52-100
    "length=10\nsteps=1\nseed=1",
    "length=10\nncars=2\nsteps=1\nseed=1\nwheels=4",
    "length=10\nncars=2\nsteps=1\nseed=1\nseed=2",
    "length=ten\nncars=2\nsteps=1\nseed=1",
    "length=10\nncars=2\nsteps=1\nseed=1\np=double",
    "length=10\nncars=2\nsteps=1\nseed=1\noutput=jpeg",
    "length=10\nncars=2\nsteps=1\nseed=1\nncar 2",
    "length=10\nncars=-2\nsteps=1\nseed=1",
    "length=10\nncars=2\nbogus=1\nsteps=1\nseed=1",
    "length=10\nncars=0\nsteps=1\nseed=1",
    "length=10\nncars=11\nsteps=1\nseed=1",
    "length=10\nncars=2\nsteps=1\nseed=1\np=1.5",
    "length=10\nncars=2\nsteps=1\nseed=1\np=nan",
    "length=10\nncars=2\nsteps=1\nseed=1\nthreads=0",
    "length=10\nncars=2\nsteps=1\nseed=1\nstride=0",
    "length=10\nncars=2\nsteps=1\nseed=1\nvmax=0",
    "length = 18446744073709551616\nncars=2\nsteps=1\nseed=1",
    " = 3\nlength=10\nncars=2\nsteps=1\nseed=1",
]
GOOD_TEXTS = [
    "length=1000\nncars=200\nsteps=1000\nseed=13",
    "# highway\n\n  length   =  100   # cells\n\tncars=4\nsteps = 10  \nseed = 5\n"
    "p = 0.25\noutput = pgm\nstride = 2\nthreads = 8\n",
    "length=10\nncars=10\nsteps=0\nseed=0\np=1\nvmax=99\noutput=ascii",
    "length=10\nncars=1\nsteps=0\nseed=0\np=1e-3",
]


def _ref_lib():
    path = os.path.join(ROOT, "oracle", "_ref", "libnasch_ref.so")
    if not os.path.exists(path):
        pytest.skip("oracle/_ref not built")
    ref = C.CDLL(path)
    ref.nasch_params_parse.argtypes = [C.c_char_p, C.POINTER(C.c_void_p), C.POINTER(C.c_uint)]
    ref.nasch_last_error.restype = C.c_char_p
    for g in ("length", "ncars", "vmax", "steps", "seed", "stride"):
        getattr(ref, "nasch_params_" + g).restype = C.c_uint64
        getattr(ref, "nasch_params_" + g).argtypes = [C.c_void_p]
    ref.nasch_params_p.restype = C.c_double
    ref.nasch_params_p.argtypes = [C.c_void_p]
    ref.nasch_params_output.argtypes = [C.c_void_p]
    return ref


@pytest.mark.parametrize("text", BAD_TEXTS + GOOD_TEXTS)
def test_parse_matches_reference(lib, text):
    ref = _ref_lib()
    ho, hr = C.c_void_p(), C.c_void_p()
    to, tr = C.c_uint(0), C.c_uint(0)
    so = lib.nasch_params_parse(text.encode(), C.byref(ho), C.byref(to))
    sr = ref.nasch_params_parse(text.encode(), C.byref(hr), C.byref(tr))
    assert so == sr
    if so:
        assert lib.nasch_last_error() == ref.nasch_last_error()
    else:
        assert to.value == tr.value
        for g in ("length", "ncars", "vmax", "p", "steps", "seed", "output", "stride"):
            assert getattr(lib, "nasch_params_" + g)(ho) == getattr(ref, "nasch_params_" + g)(hr), g


# ---- input generator -------------------------------------------------------

@pytest.mark.parametrize("L,N,vm,seed", [(1000, 200, 0, 42), (10**6, 2 * 10**5, 5, 7),
                                        (50, 50, 3, 1), (7, 1, 5, 0), (100000, 5000, 0, 3)])
def test_fill_uniform_state(L, N, vm, seed):
    x, v = nasch.fill_uniform_state(L, N, vm, seed)
    assert len(x) == N and (np.diff(x.astype(np.int64)) > 0).all() and int(x[-1]) < L
    assert int(v.max()) <= vm
    x2, v2 = nasch.fill_uniform_state(L, N, vm, seed)
    assert (x == x2).all() and (v == v2).all()
    if N == L:
        assert (x == np.arange(L)).all()
    if N >= 10000:  # roughly uniform
        assert abs(float(x.mean()) / L - 0.5) < 0.02
        if vm:
            assert abs(float(v.mean()) - vm / 2) < 0.05 * vm


# ---- integer deceleration threshold --------------------

PS = [0.0, 1e-9, 0.1, 0.13, 0.2, 0.25, 0.3, 0.4, 0.5, 0.6, 0.7, 0.9999999, 1.0,
      1 / 3, 0.123456789]


@pytest.mark.parametrize("p", PS)
def test_threshold_is_exact(lib, p):
    m = float(2147483647)
    T = lib.nasch_b200_draw_threshold(p)
    # s < T  <=>  float(s)/m < p; division is correctly rounded, so the set
    # is a prefix and checking its boundary (plus neighbours) is exhaustive.
    for s in range(max(0, T - 3), min(2147483647, T + 3) + 1):
        assert (s < T) == (float(s) / m < p), (p, T, s)


def test_threshold_exhaustive_small_modulus_argument(lib):
    """Spot-check the prefix property over a dense sample of states."""
    m = float(2147483647)
    rng = np.random.default_rng(0)
    for p in (0.13, 0.25, 0.5):
        T = lib.nasch_b200_draw_threshold(p)
        s = rng.integers(1, 2147483647, 200000)
        assert ((s < T) == (s.astype(np.float64) / m < p)).all()


def test_python_output_buffer_checks():
    """nasch.py refuses caller buffers the ABI would overrun: wrong dtype,
    too short, non-contiguous or read-only (snapshot out_x)."""
    import numpy as np
    chk = nasch._out_u64
    ok = np.zeros(10, np.uint64)
    assert chk(ok, 10, "x") is ok
    with pytest.raises(TypeError):
        chk(np.zeros(10, np.uint32), 10, "x")
    with pytest.raises(ValueError, match="holds 9"):
        chk(np.zeros(9, np.uint64), 10, "x")
    with pytest.raises(ValueError, match="contiguous"):
        chk(np.zeros(20, np.uint64)[::2], 10, "x")
    ro = np.zeros(10, np.uint64)
    ro.flags.writeable = False
    with pytest.raises(ValueError, match="writable"):
        chk(ro, 10, "x")
