"""B200-native (sm_100a) Kairos scheduling hot path.

The product is libkairos_b200.so (CUDA kernels behind the C ABI declared in
include/kairos_b200.h) plus the C++ host adapters in
include/kairos_b200.hpp. This Python package is a thin ctypes handle used by
the tests and bench.py.
"""
from ._abi import KxError, LIB_PATH, load  # noqa: F401
from .sched import (DeviceScheduler, DispatcherConfig, InstanceProfile, Profiler,  # noqa: F401
                    orchestrator_dp, record_remaining, w1_matrix)

__all__ = ["KxError", "LIB_PATH", "load", "DeviceScheduler", "DispatcherConfig",
           "InstanceProfile", "Profiler", "orchestrator_dp", "record_remaining", "w1_matrix"]
