"""Python mirror of the reference's simulation interface over the C ABI.

Class and method names follow the reference C++ types so parity tests read
like the reference's own tests:

* ``SimParams``  -- nasch::SimParams / nasch_params (src/model.hpp:16-28,
  include/nasch/nasch.h:42-78)
* ``Engine``     -- nasch::Engine / nasch_sim (src/engine.hpp:84-126,
  include/nasch/nasch.h:80-122): advance, run, steps_done, checksum,
  draws_consumed, frames, snapshot, observables

Errors surface as exceptions carrying the ABI status: ``ParamError``
(NASCH_ERR_PARSE), ``IoError`` (NASCH_ERR_IO), ``NaschError``
(NASCH_ERR_INVALID), as the reference folds its exceptions
(src/capi.cpp:27-44).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import capi as _capi

_MODES = {"none": 0, "ascii": 1, "pgm": 2}
_MODE_NAMES = {v: k for k, v in _MODES.items()}


class NaschError(RuntimeError):
    status = _capi.NASCH_ERR_INVALID


class ParamError(NaschError):
    status = _capi.NASCH_ERR_PARSE


class IoError(NaschError):
    status = _capi.NASCH_ERR_IO


def _lib():
    return _capi.load()


def _check(status: int) -> None:
    if status == _capi.NASCH_OK:
        return
    msg = _lib().nasch_last_error().decode()
    cls = {_capi.NASCH_ERR_PARSE: ParamError, _capi.NASCH_ERR_IO: IoError}.get(status, NaschError)
    raise cls(msg)


def _u64p(a):
    return a.ctypes.data_as(C.POINTER(C.c_uint64))


def _u32p(a):
    return a.ctypes.data_as(C.POINTER(C.c_uint32))


def _out_u64(a, n: int, name: str, dtype=np.uint64):
    """A caller-supplied output array must be a writable, C-contiguous u64
    (or, for the 32-bit calls, u32) vector of at least n elements: the C ABI
    writes n values through the raw pointer."""
    if not isinstance(a, np.ndarray) or a.dtype != dtype or a.ndim != 1:
        raise TypeError(f"{name} must be a 1-D numpy {np.dtype(dtype).name} array")
    if not a.flags.c_contiguous or not a.flags.writeable:
        raise ValueError(f"{name} must be C-contiguous and writable")
    if len(a) < n:
        raise ValueError(f"{name} holds {len(a)} values; the ring has {n} cars")
    return a


class SimParams:
    """Owned nasch_params handle (defaults vmax=5, p=0.13, output none)."""

    def __init__(self, length: int = 0, ncars: int = 0, vmax: int = 5, p: float = 0.13,
                 steps: int = 0, seed: int = 0, output: str = "none", stride: int = 1,
                 *, _handle=None):
        lib = _lib()
        if _handle is None:
            h = C.c_void_p()
            _check(lib.nasch_params_new(C.byref(h)))
            self._h = h
            self.length, self.ncars, self.vmax, self.p = length, ncars, vmax, p
            self.steps, self.seed, self.output, self.stride = steps, seed, output, stride
        else:
            self._h = _handle

    @classmethod
    def parse(cls, text: str) -> tuple["SimParams", int]:
        h, threads = C.c_void_p(), C.c_uint(0)
        _check(_lib().nasch_params_parse(text.encode(), C.byref(h), C.byref(threads)))
        return cls(_handle=h), threads.value

    @classmethod
    def load(cls, path: str) -> tuple["SimParams", int]:
        h, threads = C.c_void_p(), C.c_uint(0)
        _check(_lib().nasch_params_load(str(path).encode(), C.byref(h), C.byref(threads)))
        return cls(_handle=h), threads.value

    def validate(self) -> None:
        _check(_lib().nasch_params_validate(self._h))

    def _set(self, name, value):
        _check(getattr(_lib(), "nasch_params_set_" + name)(self._h, value))

    def _get(self, name):
        return getattr(_lib(), "nasch_params_" + name)(self._h)

    length = property(lambda s: s._get("length"), lambda s, v: s._set("length", v))
    ncars = property(lambda s: s._get("ncars"), lambda s, v: s._set("ncars", v))
    vmax = property(lambda s: s._get("vmax"), lambda s, v: s._set("vmax", v))
    p = property(lambda s: s._get("p"), lambda s, v: s._set("p", float(v)))
    steps = property(lambda s: s._get("steps"), lambda s, v: s._set("steps", v))
    seed = property(lambda s: s._get("seed"), lambda s, v: s._set("seed", v))
    stride = property(lambda s: s._get("stride"), lambda s, v: s._set("stride", v))
    output = property(lambda s: _MODE_NAMES[s._get("output")],
                      lambda s, v: s._set("output", _MODES[v]))

    def close(self):
        if getattr(self, "_h", None):
            _lib().nasch_params_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Engine:
    """A simulation on the B200 engine (nasch_sim)."""

    AGENT, GRID_REFERENCE, CUDA = 0, 1, 2

    def __init__(self, params: SimParams, workers: int = 1, kind: int = 0, *, _handle=None):
        if _handle is None:
            h = C.c_void_p()
            _check(_lib().nasch_sim_new_kind(params._h, workers, kind, C.byref(h)))
        else:
            h = _handle
        self._h = h
        self.ncars = params.ncars
        self.length = params.length

    @classmethod
    def distributed(cls, params: SimParams, rank: int, world: int, nccl_id: bytes) -> "Engine":
        """One segment of a ring split over `world` processes (one GPU each),
        exchanging through NCCL; `nccl_id` comes from nccl_unique_id() on
        rank 0."""
        buf = C.create_string_buffer(bytes(nccl_id), 128)
        h = C.c_void_p()
        _check(_lib().nasch_sim_new_distributed(params._h, rank, world, buf, C.byref(h)))
        return cls(params, _handle=h)

    def shard_range(self) -> tuple[int, int]:
        first, count = C.c_uint64(), C.c_uint64()
        _check(_lib().nasch_sim_shard_range(self._h, C.byref(first), C.byref(count)))
        return first.value, count.value

    # -- stepping ------------------------------------------------------
    def advance(self, steps: int) -> None:
        _check(_lib().nasch_sim_advance(self._h, steps))

    def run(self) -> None:
        _check(_lib().nasch_sim_run(self._h))

    def enqueue(self, steps: int) -> None:
        _check(_lib().nasch_sim_enqueue(self._h, steps))

    def synchronize(self) -> None:
        _check(_lib().nasch_sim_synchronize(self._h))

    # -- accessors -------------------------------------------------------
    @property
    def steps_done(self) -> int:
        return _lib().nasch_sim_steps_done(self._h)

    @property
    def checksum(self) -> int:
        return _lib().nasch_sim_checksum(self._h)

    @property
    def draws_consumed(self) -> int:
        return _lib().nasch_sim_draws(self._h)

    @property
    def frame_count(self) -> int:
        return _lib().nasch_sim_frame_count(self._h)

    @property
    def kernel_launches(self) -> int:
        return _lib().nasch_sim_kernel_launches(self._h)

    @property
    def steps_per_launch(self) -> int:
        return _lib().nasch_sim_steps_per_launch(self._h)

    @property
    def exchange_mode(self) -> int:
        """0 one segment, 1 collective exchange, 2 peer-memory exchange."""
        return _lib().nasch_sim_exchange_mode(self._h)

    @property
    def cuda_stream(self) -> int:
        return _lib().nasch_sim_cuda_stream(self._h) or 0

    def set_checksum(self, enabled: bool) -> None:
        _check(_lib().nasch_sim_set_checksum(self._h, 1 if enabled else 0))

    def snapshot(self, *, out_x=None, out_v=None):
        """Current (positions, velocities) in increasing-position order."""
        x = np.empty(self.ncars, np.uint64) if out_x is None else _out_u64(out_x, self.ncars, "out_x")
        v = np.empty(self.ncars, np.uint64) if out_v is None else _out_u64(out_v, self.ncars, "out_v")
        _check(_lib().nasch_sim_state(self._h, _u64p(x), _u64p(v), min(len(x), len(v))))
        return x, v

    def snapshot32(self, *, out_x=None, out_v=None):
        """The same snapshot as u32 arrays (BASELINE's int32 state format,
        nasch_sim_state32): positions reach a page-locked out_x by DMA."""
        x = np.empty(self.ncars, np.uint32) if out_x is None else _out_u64(out_x, self.ncars, "out_x", np.uint32)
        v = np.empty(self.ncars, np.uint32) if out_v is None else _out_u64(out_v, self.ncars, "out_v", np.uint32)
        _check(_lib().nasch_sim_state32(self._h, _u32p(x), _u32p(v), min(len(x), len(v))))
        return x, v

    def job32(self, x, v, steps: int, *, out_x=None, out_v=None):
        """set_state(x, v) + advance(steps) + snapshot32() in one call
        (nasch_sim_job32): u32 input, u32 output; streamed (upload, steps
        and download overlapped) for page-locked arrays within one K-step
        launch."""
        x = np.ascontiguousarray(x)
        v = np.ascontiguousarray(v)
        if x.dtype != np.uint32 or v.dtype != np.uint32 or x.ndim != 1 or v.ndim != 1 or len(x) != len(v):
            raise ValueError("job32 takes 1-D uint32 positions and velocities of equal length")
        ox = np.empty(self.ncars, np.uint32) if out_x is None else _out_u64(out_x, self.ncars, "out_x", np.uint32)
        ov = np.empty(self.ncars, np.uint32) if out_v is None else _out_u64(out_v, self.ncars, "out_v", np.uint32)
        _check(_lib().nasch_sim_job32(self._h, _u32p(x), _u32p(v), len(x), steps, _u32p(ox), _u32p(ov),
                                      min(len(ox), len(ov))))
        return ox, ov

    def snapshot_async(self, out_x, out_v) -> None:
        """Start a snapshot into (out_x, out_v) (u64, length ncars) that
        completes while the caller advances; call snapshot_wait() before
        reading the arrays (nasch_sim_state_async)."""
        _out_u64(out_x, self.ncars, "out_x")
        _out_u64(out_v, self.ncars, "out_v")
        self._pending = (out_x, out_v)  # keep the buffers alive
        _check(_lib().nasch_sim_state_async(self._h, _u64p(out_x), _u64p(out_v),
                                            min(len(out_x), len(out_v))))

    def segment_snapshot(self, *, out_x=None, out_v=None):
        """The cars this process holds (shard_range), widened to u64:
        (x, v, first_rank) with element k at rank (first_rank + k) mod N
        (nasch_sim_state_segment; not a collective call).  A sim holding the
        whole ring returns it in rank order with first_rank 0."""
        _, count = self.shard_range()
        x = np.empty(count, np.uint64) if out_x is None else _out_u64(out_x, count, "out_x")
        v = np.empty(count, np.uint64) if out_v is None else _out_u64(out_v, count, "out_v")
        first = C.c_uint64()
        _check(_lib().nasch_sim_state_segment(self._h, _u64p(x), _u64p(v), min(len(x), len(v)),
                                              C.byref(first)))
        return x, v, first.value

    def segment_snapshot32(self, *, out_x=None, out_v=None):
        """segment_snapshot into u32 arrays (nasch_sim_state_segment32)."""
        _, count = self.shard_range()
        x = np.empty(count, np.uint32) if out_x is None else _out_u64(out_x, count, "out_x", np.uint32)
        v = np.empty(count, np.uint32) if out_v is None else _out_u64(out_v, count, "out_v", np.uint32)
        first = C.c_uint64()
        _check(_lib().nasch_sim_state_segment32(self._h, _u32p(x), _u32p(v), min(len(x), len(v)),
                                                C.byref(first)))
        return x, v, first.value

    def segment_snapshot_async(self, out_x, out_v) -> int:
        """Start a segment snapshot into (out_x, out_v); returns first_rank.
        The arrays are complete after snapshot_wait()."""
        _, count = self.shard_range()
        _out_u64(out_x, count, "out_x")
        _out_u64(out_v, count, "out_v")
        self._pending = (out_x, out_v)
        first = C.c_uint64()
        _check(_lib().nasch_sim_state_segment_async(self._h, _u64p(out_x), _u64p(out_v),
                                                    min(len(out_x), len(out_v)), C.byref(first)))
        return first.value

    def set_segment_state(self, x, v) -> None:
        """Collective set_state from this process's segment of the new
        rank-ordered state (nasch_sim_set_state_segment)."""
        x = np.ascontiguousarray(x, np.uint64)
        v = np.ascontiguousarray(v, np.uint64)
        if x.ndim != 1 or v.ndim != 1 or len(x) != len(v):
            raise ValueError(f"positions and velocities must be 1-D of equal length "
                             f"(got {x.shape} and {v.shape})")
        _check(_lib().nasch_sim_set_state_segment(self._h, _u64p(x), _u64p(v), len(x)))

    def snapshot_wait(self) -> None:
        _check(_lib().nasch_sim_state_wait(self._h))
        self._pending = None

    def observables(self) -> tuple[float, float, float]:
        """(density, mean_velocity, flow) as nasch_sim_observables."""
        d, m, f = C.c_double(), C.c_double(), C.c_double()
        _check(_lib().nasch_sim_observables(self._h, C.byref(d), C.byref(m), C.byref(f)))
        return d.value, m.value, f.value

    def set_state(self, x, v) -> None:
        x = np.ascontiguousarray(x)
        v = np.ascontiguousarray(v)
        if x.ndim != 1 or v.ndim != 1 or len(x) != len(v):
            raise ValueError(f"positions and velocities must be 1-D of equal length "
                             f"(got {x.shape} and {v.shape})")
        if x.dtype == np.uint32 and v.dtype == np.uint32:
            _check(_lib().nasch_sim_set_state32(self._h, _u32p(x), _u32p(v), len(x)))
        else:
            x = np.ascontiguousarray(x, np.uint64)
            v = np.ascontiguousarray(v, np.uint64)
            _check(_lib().nasch_sim_set_state(self._h, _u64p(x), _u64p(v), len(x)))

    def _series(self, fn, dtype, ptr):
        n = C.c_size_t()
        _check(fn(self._h, None, 0, C.byref(n)))
        out = np.empty(n.value, dtype)
        _check(fn(self._h, ptr(out), n.value, C.byref(n)))
        return out

    def sumv_series(self) -> np.ndarray:
        return self._series(_lib().nasch_sim_sumv_series, np.uint64, _u64p)

    def wrap_series(self) -> np.ndarray:
        return self._series(_lib().nasch_sim_wrap_series, np.uint64, _u64p)

    def mean_velocity_series(self) -> np.ndarray:
        return self._series(_lib().nasch_sim_mean_velocity_series, np.float64,
                            lambda a: a.ctypes.data_as(C.POINTER(C.c_double)))

    def write_ascii(self, path: str) -> None:
        _check(_lib().nasch_sim_write_ascii(self._h, str(path).encode()))

    def write_pgm(self, path: str) -> None:
        _check(_lib().nasch_sim_write_pgm(self._h, str(path).encode()))

    def close(self):
        if getattr(self, "_h", None):
            _lib().nasch_sim_free(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Ensemble:
    """Many independent rings advanced together (nasch_ensemble)."""

    def __init__(self, params: list[SimParams]):
        self._params = list(params)  # keep handles alive during construction
        arr = (C.c_void_p * len(params))(*[p._h.value for p in params])
        h = C.c_void_p()
        _check(_lib().nasch_ensemble_new(arr, len(params), C.byref(h)))
        self._h = h
        self.ncars = [p.ncars for p in params]
        self.length = [p.length for p in params]

    def __len__(self):
        return _lib().nasch_ensemble_size(self._h)

    def set_state(self, ring: int, x, v) -> None:
        x = np.ascontiguousarray(x, np.uint32)
        v = np.ascontiguousarray(v, np.uint32)
        if x.ndim != 1 or v.ndim != 1 or len(x) != len(v):
            raise ValueError(f"positions and velocities must be 1-D of equal length "
                             f"(got {x.shape} and {v.shape})")
        _check(_lib().nasch_ensemble_set_state32(self._h, ring, _u32p(x), _u32p(v), len(x)))

    def set_state_all(self, x, v) -> None:
        """Every ring at once: rank-ordered rings concatenated in ring order
        (nasch_ensemble_set_state_all32)."""
        x = np.ascontiguousarray(x, np.uint32)
        v = np.ascontiguousarray(v, np.uint32)
        if x.ndim != 1 or v.ndim != 1 or len(x) != len(v):
            raise ValueError(f"positions and velocities must be 1-D of equal length "
                             f"(got {x.shape} and {v.shape})")
        _check(_lib().nasch_ensemble_set_state_all32(self._h, _u32p(x), _u32p(v), len(x)))

    def advance(self, steps: int) -> None:
        _check(_lib().nasch_ensemble_advance(self._h, steps))

    def enqueue(self, steps: int) -> None:
        _check(_lib().nasch_ensemble_enqueue(self._h, steps))

    def synchronize(self) -> None:
        _check(_lib().nasch_ensemble_synchronize(self._h))

    def steps_done(self, ring: int) -> int:
        return _lib().nasch_ensemble_steps_done(self._h, ring)

    def sumv_totals(self) -> np.ndarray:
        out = np.empty(len(self.ncars), np.uint64)
        _check(_lib().nasch_ensemble_sumv_totals(self._h, _u64p(out), len(out)))
        return out

    def sumv_last(self) -> np.ndarray:
        out = np.empty(len(self.ncars), np.uint64)
        _check(_lib().nasch_ensemble_sumv_last(self._h, _u64p(out), len(out)))
        return out

    def snapshot(self, ring: int):
        n = self.ncars[ring]
        x = np.empty(n, np.uint64)
        v = np.empty(n, np.uint64)
        _check(_lib().nasch_ensemble_state(self._h, ring, _u64p(x), _u64p(v), n))
        return x, v

    @property
    def cuda_stream(self) -> int:
        return _lib().nasch_ensemble_cuda_stream(self._h) or 0

    @property
    def kernel_launches(self) -> int:
        return _lib().nasch_ensemble_kernel_launches(self._h)

    def close(self):
        if getattr(self, "_h", None):
            _lib().nasch_ensemble_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def fill_uniform_state(length: int, ncars: int, vmax_init: int, seed: int):
    """BASELINE inputs: sorted distinct uniform positions (u32) and
    velocities uniform in [0, vmax_init] (u32)."""
    x = np.empty(ncars, np.uint32)
    v = np.empty(ncars, np.uint32)
    _check(_lib().nasch_fill_uniform_state(length, ncars, vmax_init, seed, _u32p(x), _u32p(v)))
    return x, v


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(_lib().nasch_nccl_unique_id(buf))
    return buf.raw


def physical_cores() -> int:
    return _lib().nasch_physical_cores()


def partition_rings(ncars, world: int):
    """Contiguous ring ranges for `world` ranks, balanced by total cars
    (an ensemble shards with no communication while
    stepping; N varies 10x across a density sweep, so equal ring counts would
    not balance).  Returns [(lo, hi)] per rank; every ring in exactly one."""
    n = np.asarray(ncars, dtype=np.int64)
    if world < 1:
        raise ValueError("world must be >= 1")
    csum = np.concatenate([[0], np.cumsum(n)])
    total = int(csum[-1])
    cuts = [0]
    for r in range(1, world):
        # first ring whose start reaches r/world of the cars
        cuts.append(int(np.searchsorted(csum, (total * r + world - 1) // world, side="left")))
    cuts.append(len(n))
    cuts = [min(max(c, cuts[i - 1] if i else 0), len(n)) for i, c in enumerate(cuts)]
    return [(cuts[r], cuts[r + 1]) for r in range(world)]
