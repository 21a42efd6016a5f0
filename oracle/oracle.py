"""ctypes wrappers for the parity checkers.  TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` leg may import this module.  The product
(paper_2309_14311_b200) never does; its CUDA path fails loudly when its
own extension is missing instead of falling back here.

Two checkers:

* ``Port``  -- oracle/_build/libnasch_oracle.so, our plain-C restatement of
  the reference hot path (oracle/nasch_oracle.c, each function citing the
  reference file:line it restates).
* ``Ref``   -- oracle/_ref/libnasch_ref.so, the reference sources compiled
  unmodified (oracle/Makefile) plus ref_harness.cpp; runs the reference's
  own OpenMP Engine, optionally on injected initial state.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "_build", "libnasch_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libnasch_ref.so")

M = 2147483647
A = 48271
FNV_BASIS = 14695981039346656037

_u64p = C.POINTER(C.c_uint64)
_i64p = C.POINTER(C.c_int64)


def build() -> None:
    """Compile the C restatement (and oracle/_ref when the reference
    sources are present).  Building the checker is not using it."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _ptr(a):
    return a.ctypes.data_as(_u64p) if a is not None else None


class Port:
    """Our C restatement of the reference path (oracle/nasch_oracle.c)."""

    def __init__(self, path: str = PORT_SO):
        if not os.path.exists(path):
            build()
        lib = C.CDLL(path)
        lib.or_lcg_seeded.argtypes = [C.c_uint64]
        lib.or_lcg_seeded.restype = C.c_uint64
        lib.or_lcg_next.argtypes = [_u64p]
        lib.or_lcg_next.restype = C.c_uint64
        lib.or_uniform01.argtypes = [_u64p]
        lib.or_uniform01.restype = C.c_double
        lib.or_jump_coefficients.argtypes = [C.c_uint64, _u64p, _u64p]
        lib.or_lcg_jump.argtypes = [C.c_uint64, C.c_uint64]
        lib.or_lcg_jump.restype = C.c_uint64
        lib.or_init_state.argtypes = [C.c_uint64, C.c_uint64, _u64p, _u64p]
        lib.or_gap_ahead.argtypes = [_u64p, C.c_size_t, C.c_uint64, C.c_size_t]
        lib.or_gap_ahead.restype = C.c_uint64
        lib.or_step_serial.argtypes = [_u64p, _u64p, C.c_size_t, C.c_uint64,
                                       C.c_uint64, C.c_double, _u64p, _u64p]
        lib.or_step_serial.restype = C.c_size_t
        lib.or_step_grid_serial.argtypes = [_i64p, C.c_uint64, C.c_uint64,
                                            C.c_double, _u64p]
        lib.or_fnv1a64_value.argtypes = [C.c_uint64, C.c_uint64]
        lib.or_fnv1a64_value.restype = C.c_uint64
        lib.or_hash_row.argtypes = [C.c_uint64, _u64p, _u64p, C.c_size_t]
        lib.or_hash_row.restype = C.c_uint64
        lib.or_mean_velocity.argtypes = [_u64p, C.c_size_t]
        lib.or_mean_velocity.restype = C.c_double
        lib.or_run.argtypes = [C.c_uint64, C.c_uint64, C.c_double, _u64p,
                               C.c_uint64, _u64p, _u64p, C.c_size_t, _u64p,
                               _u64p, _u64p]
        lib.or_run.restype = C.c_int
        _u32p = C.POINTER(C.c_uint32)
        lib.or_fill_uniform_state.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64,
                                              C.c_uint64, _u32p, _u32p]
        lib.or_fill_uniform_state.restype = C.c_int
        self.lib = lib

    # -- PRNG ------------------------------------------------------------
    def seeded(self, seed: int) -> int:
        return self.lib.or_lcg_seeded(seed)

    def next(self, state: int) -> tuple[int, int]:
        s = C.c_uint64(state)
        r = self.lib.or_lcg_next(C.byref(s))
        return r, s.value

    def uniform01(self, state: int) -> tuple[float, int]:
        s = C.c_uint64(state)
        u = self.lib.or_uniform01(C.byref(s))
        return u, s.value

    def jump(self, state: int, k: int) -> int:
        return self.lib.or_lcg_jump(state, k)

    def jump_coefficients(self, k: int) -> tuple[int, int]:
        mul, add = C.c_uint64(), C.c_uint64()
        self.lib.or_jump_coefficients(k, C.byref(mul), C.byref(add))
        return mul.value, add.value

    # -- BASELINE input generator (not a reference function) ----------------
    def fill_uniform_state(self, L: int, N: int, vmax_init: int, seed: int):
        """Seeded uniform distinct sorted positions and velocities in
        [0, vmax_init], both u32 -- the same inputs nasch_fill_uniform_state
        gives the GPU arm (tests/test_oracle.py checks equality)."""
        x = np.empty(N, np.uint32)
        v = np.empty(N, np.uint32)
        u32 = C.POINTER(C.c_uint32)
        rc = self.lib.or_fill_uniform_state(L, N, vmax_init, seed, x.ctypes.data_as(u32),
                                            v.ctypes.data_as(u32))
        if rc:
            raise ValueError("need N <= L < 2^32")
        return x, v

    # -- model -----------------------------------------------------------
    def init_state(self, L: int, N: int):
        x = np.empty(N, np.uint64)
        v = np.empty(N, np.uint64)
        self.lib.or_init_state(L, N, _ptr(x), _ptr(v))
        return x, v

    def gap_ahead(self, x, L: int, i: int) -> int:
        x = np.ascontiguousarray(x, np.uint64)
        return self.lib.or_gap_ahead(_ptr(x), len(x), L, i)

    def step(self, x, v, L, vmax, p, rng_state):
        """One step in place; returns (wrapped, new rng state)."""
        s = C.c_uint64(rng_state)
        tmp = np.empty(max(len(x), 1), np.uint64)
        w = self.lib.or_step_serial(_ptr(x), _ptr(v), len(x), L, vmax, p,
                                    C.byref(s), _ptr(tmp))
        return w, s.value

    def step_grid(self, cells, L, vmax, p, rng_state):
        s = C.c_uint64(rng_state)
        self.lib.or_step_grid_serial(cells.ctypes.data_as(_i64p), L, vmax, p,
                                     C.byref(s))
        return s.value

    def fnv_value(self, h: int, value: int) -> int:
        return self.lib.or_fnv1a64_value(h, value)

    def hash_row(self, h: int, x, v) -> int:
        x = np.ascontiguousarray(x, np.uint64)
        v = np.ascontiguousarray(v, np.uint64)
        return self.lib.or_hash_row(h, _ptr(x), _ptr(v), len(x))

    def run(self, L, vmax, p, seed, steps, x, v, *, rng_state=None,
            checksum=FNV_BASIS, want_checksum=True):
        """Runs `steps` steps from rank-ordered (x, v) (copied).  Returns
        dict(x, v, sumv, wraps, checksum, rng)."""
        x = np.array(x, np.uint64, copy=True)
        v = np.array(v, np.uint64, copy=True)
        s = C.c_uint64(self.seeded(seed) if rng_state is None else rng_state)
        sumv = np.empty(max(steps, 1), np.uint64)
        wraps = np.empty(max(steps, 1), np.uint64)
        h = C.c_uint64(checksum)
        rc = self.lib.or_run(L, vmax, p, C.byref(s), steps, _ptr(x), _ptr(v),
                             len(x), _ptr(sumv), _ptr(wraps),
                             C.byref(h) if want_checksum else None)
        assert rc == 0
        return dict(x=x, v=v, sumv=sumv[:steps], wraps=wraps[:steps],
                    checksum=h.value if want_checksum else None, rng=s.value)


class Ref:
    """The reference implementation itself (oracle/_ref/libnasch_ref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            build()
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        lib = C.CDLL(path)
        lib.refh_run.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.c_double,
                                 C.c_uint64, C.c_uint64, C.c_uint, _u64p, _u64p,
                                 C.c_int, _u64p, _u64p, _u64p, _u64p, _u64p,
                                 C.POINTER(C.c_double)]
        lib.refh_run.restype = C.c_int
        lib.refh_last_error.restype = C.c_char_p
        lib.refh_physical_cores.restype = C.c_uint
        self.lib = lib

    def physical_cores(self) -> int:
        return self.lib.refh_physical_cores()

    def run(self, L, N, vmax, p, seed, steps, *, workers=1, x0=None, v0=None,
            per_step=True, want_state=True):
        """Returns dict(x, v, sumv, wraps, checksum, seconds); sumv / wraps
        (per-step velocity sums and crossing counts) only with per_step."""
        x0 = None if x0 is None else np.ascontiguousarray(x0, np.uint64)
        v0 = None if v0 is None else np.ascontiguousarray(v0, np.uint64)
        x = np.empty(N, np.uint64) if want_state else None
        v = np.empty(N, np.uint64) if want_state else None
        sumv = np.empty(max(steps, 1), np.uint64) if per_step else None
        wraps = np.empty(max(steps, 1), np.uint64) if per_step else None
        h = C.c_uint64()
        sec = C.c_double()
        rc = self.lib.refh_run(L, N, vmax, p, seed, steps, workers, _ptr(x0),
                               _ptr(v0), 1 if per_step else 0, _ptr(x),
                               _ptr(v), _ptr(sumv), _ptr(wraps), C.byref(h), C.byref(sec))
        if rc != 0:
            raise RuntimeError(self.lib.refh_last_error().decode())
        return dict(x=x, v=v, sumv=None if sumv is None else sumv[:steps],
                    wraps=None if wraps is None else wraps[:steps],
                    checksum=h.value, seconds=sec.value)
