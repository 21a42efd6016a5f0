"""ctypes binding of libnasch_b200.so (include/nasch/nasch.h).

This is the same C ABI the reference exports from libnasch.so
(/root/reference/proj/include/nasch/nasch.h:40-127) plus the B200
extensions; ``INTEGRATION.md`` shows the equivalent binding a reference
caller would write.  The library is built in-tree by ``build()``; loading
fails loudly if it is missing -- there is no fallback implementation.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libnasch_b200.so")
CSRC = os.path.join(PKG, "csrc")

NASCH_OK, NASCH_ERR_INVALID, NASCH_ERR_PARSE, NASCH_ERR_IO = 0, 1, 2, 3
NASCH_OUTPUT_NONE, NASCH_OUTPUT_ASCII, NASCH_OUTPUT_PGM = 0, 1, 2
NASCH_ENGINE_AGENT, NASCH_ENGINE_GRID_REFERENCE, NASCH_ENGINE_CUDA = 0, 1, 2

# name -> (restype, argtypes); every symbol include/nasch/nasch.h declares.
_P = C.c_void_p
_u64 = C.c_uint64
_u64p = C.POINTER(C.c_uint64)
_u32p = C.POINTER(C.c_uint32)
_dp = C.POINTER(C.c_double)
_szp = C.POINTER(C.c_size_t)
SIGNATURES: dict[str, tuple] = {
    # reference ABI (36 symbols)
    "nasch_last_error": (C.c_char_p, []),
    "nasch_params_new": (C.c_int, [C.POINTER(_P)]),
    "nasch_params_parse": (C.c_int, [C.c_char_p, C.POINTER(_P), C.POINTER(C.c_uint)]),
    "nasch_params_load": (C.c_int, [C.c_char_p, C.POINTER(_P), C.POINTER(C.c_uint)]),
    "nasch_params_free": (None, [_P]),
    "nasch_params_set_length": (C.c_int, [_P, _u64]),
    "nasch_params_set_ncars": (C.c_int, [_P, _u64]),
    "nasch_params_set_vmax": (C.c_int, [_P, _u64]),
    "nasch_params_set_p": (C.c_int, [_P, C.c_double]),
    "nasch_params_set_steps": (C.c_int, [_P, _u64]),
    "nasch_params_set_seed": (C.c_int, [_P, _u64]),
    "nasch_params_set_output": (C.c_int, [_P, C.c_int]),
    "nasch_params_set_stride": (C.c_int, [_P, _u64]),
    "nasch_params_length": (_u64, [_P]),
    "nasch_params_ncars": (_u64, [_P]),
    "nasch_params_vmax": (_u64, [_P]),
    "nasch_params_p": (C.c_double, [_P]),
    "nasch_params_steps": (_u64, [_P]),
    "nasch_params_seed": (_u64, [_P]),
    "nasch_params_output": (C.c_int, [_P]),
    "nasch_params_stride": (_u64, [_P]),
    "nasch_params_validate": (C.c_int, [_P]),
    "nasch_sim_new": (C.c_int, [_P, C.c_uint, C.POINTER(_P)]),
    "nasch_sim_new_kind": (C.c_int, [_P, C.c_uint, C.c_int, C.POINTER(_P)]),
    "nasch_sim_free": (None, [_P]),
    "nasch_sim_advance": (C.c_int, [_P, _u64]),
    "nasch_sim_run": (C.c_int, [_P]),
    "nasch_sim_steps_done": (_u64, [_P]),
    "nasch_sim_checksum": (_u64, [_P]),
    "nasch_sim_draws": (_u64, [_P]),
    "nasch_sim_frame_count": (_u64, [_P]),
    "nasch_sim_observables": (C.c_int, [_P, _dp, _dp, _dp]),
    "nasch_sim_state": (C.c_int, [_P, _u64p, _u64p, C.c_size_t]),
    "nasch_sim_write_ascii": (C.c_int, [_P, C.c_char_p]),
    "nasch_sim_write_pgm": (C.c_int, [_P, C.c_char_p]),
    "nasch_physical_cores": (C.c_uint, []),
    # B200 extensions
    "nasch_sim_set_state": (C.c_int, [_P, _u64p, _u64p, C.c_size_t]),
    "nasch_sim_state_async": (C.c_int, [_P, _u64p, _u64p, C.c_size_t]),
    "nasch_sim_state_wait": (C.c_int, [_P]),
    "nasch_sim_set_state32": (C.c_int, [_P, _u32p, _u32p, C.c_size_t]),
    "nasch_sim_set_checksum": (C.c_int, [_P, C.c_int]),
    "nasch_sim_sumv_series": (C.c_int, [_P, _u64p, C.c_size_t, _szp]),
    "nasch_sim_mean_velocity_series": (C.c_int, [_P, _dp, C.c_size_t, _szp]),
    "nasch_sim_wrap_series": (C.c_int, [_P, _u64p, C.c_size_t, _szp]),
    "nasch_sim_enqueue": (C.c_int, [_P, _u64]),
    "nasch_sim_synchronize": (C.c_int, [_P]),
    "nasch_sim_cuda_stream": (C.c_void_p, [_P]),
    "nasch_sim_kernel_launches": (_u64, [_P]),
    "nasch_sim_steps_per_launch": (C.c_uint, [_P]),
    "nasch_sim_exchange_mode": (C.c_uint, [_P]),
    "nasch_fill_uniform_state": (C.c_int, [_u64, _u64, _u64, _u64, _u32p, _u32p]),
    "nasch_b200_version": (C.c_char_p, []),
    "nasch_b200_draw_threshold": (C.c_uint32, [C.c_double]),
    # multi-GPU ring
    "nasch_nccl_unique_id": (C.c_int, [C.c_void_p]),
    "nasch_sim_new_distributed": (C.c_int, [_P, C.c_uint, C.c_uint, C.c_void_p, C.POINTER(_P)]),
    "nasch_sim_shard_range": (C.c_int, [_P, _u64p, _u64p]),
    "nasch_sim_state_segment": (C.c_int, [_P, _u64p, _u64p, C.c_size_t, _u64p]),
    "nasch_sim_state_segment32": (C.c_int, [_P, _u32p, _u32p, C.c_size_t, _u64p]),
    "nasch_sim_state32": (C.c_int, [_P, _u32p, _u32p, C.c_size_t]),
    "nasch_sim_job32": (C.c_int, [_P, _u32p, _u32p, C.c_size_t, _u64, _u32p, _u32p, C.c_size_t]),
    "nasch_sim_state_segment_async": (C.c_int, [_P, _u64p, _u64p, C.c_size_t, _u64p]),
    "nasch_sim_set_state_segment": (C.c_int, [_P, _u64p, _u64p, C.c_size_t]),
    # ensembles
    "nasch_ensemble_new": (C.c_int, [C.POINTER(_P), C.c_size_t, C.POINTER(_P)]),
    "nasch_ensemble_free": (None, [_P]),
    "nasch_ensemble_size": (C.c_size_t, [_P]),
    "nasch_ensemble_set_state32": (C.c_int, [_P, C.c_size_t, _u32p, _u32p, C.c_size_t]),
    "nasch_ensemble_set_state_all32": (C.c_int, [_P, _u32p, _u32p, C.c_size_t]),
    "nasch_ensemble_advance": (C.c_int, [_P, _u64]),
    "nasch_ensemble_enqueue": (C.c_int, [_P, _u64]),
    "nasch_ensemble_synchronize": (C.c_int, [_P]),
    "nasch_ensemble_steps_done": (_u64, [_P, C.c_size_t]),
    "nasch_ensemble_sumv_totals": (C.c_int, [_P, _u64p, C.c_size_t]),
    "nasch_ensemble_sumv_last": (C.c_int, [_P, _u64p, C.c_size_t]),
    "nasch_ensemble_state": (C.c_int, [_P, C.c_size_t, _u64p, _u64p, C.c_size_t]),
    "nasch_ensemble_cuda_stream": (C.c_void_p, [_P]),
    "nasch_ensemble_kernel_launches": (_u64, [_P]),
}
REFERENCE_SYMBOLS = list(SIGNATURES)[:36]

_lib = None


def build(verbose: bool = False) -> None:
    """Compile libnasch_b200.so in-tree (sm_100a)."""
    out = None if verbose else subprocess.DEVNULL
    subprocess.run(["make", "-s", "-C", CSRC], check=True, stdout=out)


def load(path: str = LIB_PATH):
    """Load the library once and attach signatures.  Raises if absent.
    NASCH_B200_LIB overrides the path (kernel-geometry experiments)."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("NASCH_B200_LIB") or path
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build it with `make -C {CSRC}` "
            "(the B200 engine has no fallback implementation)")
    lib = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib
