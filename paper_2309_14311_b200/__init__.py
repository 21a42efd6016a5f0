"""B200-native NaSch traffic engine (drop-in for the reference's C ABI).

The product is ``libnasch_b200.so`` (C ABI in include/nasch/nasch.h, host
C++ + sm_100a CUDA in csrc/).  This package only builds and binds it.
"""
from .capi import build, load, LIB_PATH  # noqa: F401
from .nasch import (  # noqa: F401
    Engine,
    Ensemble,
    IoError,
    NaschError,
    ParamError,
    SimParams,
    fill_uniform_state,
    physical_cores,
)
