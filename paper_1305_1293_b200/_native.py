"""ctypes binding of the C ABI in include/pch_b200.h (libpch_b200.so).

The library is built in-tree by ``paper_1305_1293_b200.build`` (nvcc,
sm_100a).  There is no fallback: if the library is missing or no CUDA
device is visible, every solve raises ``NativeUnavailable``.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PCH_B200_LIB") or os.path.join(_HERE, "_lib", "libpch_b200.so")

ABI_VERSION = 3

PCH_OK = 0
PCH_ERR_CUDA = 1
PCH_ERR_SOURCE = 2
PCH_ERR_CONFIG = 3
PCH_ERR_GUARD = 4
PCH_ERR_MESH = 5
PCH_ERR_NOMEM = 6

FLAG_NO_RECHECK = 1
FLAG_DETERMINISTIC = 2
FLAG_ABSOLUTE_TINY = 4
FLAG_PHASE_TIMES = 8
FLAG_DEDUPE = 16


class NativeUnavailable(RuntimeError):
    """The CUDA library is not built or cannot be loaded."""


class PchConfig(ctypes.Structure):
    _fields_ = [("k", ctypes.c_int64), ("selection_mode", ctypes.c_int32),
                ("fan_mode", ctypes.c_int32), ("epsilon_window", ctypes.c_double),
                ("max_iterations", ctypes.c_int64),
                ("pool_capacity", ctypes.c_int64), ("flags", ctypes.c_int32),
                ("chain", ctypes.c_int32), ("time_limit_s", ctypes.c_double),
                ("fan_margin", ctypes.c_double)]


STAT_FIELDS = ("iterations", "windows_propagated", "total_windows_created",
               "total_windows_pruned", "pruned_ich", "pruned_split",
               "pruned_tiny", "pruned_degenerate", "pruned_duplicate",
               "pruned_recheck", "windows_stored", "max_children_per_window",
               "events_created", "events_applied", "peak_active_pool",
               "fans_emitted", "buffer_regrows", "pool_restarts", "grid_barriers")


TIME_FIELDS = ("time_total_ms", "time_kernel_ms", "time_select_ms",
               "time_propagate_ms", "time_compact_ms", "time_events_ms",
               "prop_item_us")


class PchStats(ctypes.Structure):
    _fields_ = ([(f, ctypes.c_int64) for f in STAT_FIELDS]
                + [(f, ctypes.c_double) for f in TIME_FIELDS])


# symbols declared in include/pch_b200.h
EXPORTS = ("pch_abi_version", "pch_last_error", "pch_device_count",
           "pch_mesh_create", "pch_mesh_destroy", "pch_mesh_device_bytes",
           "pch_run", "pch_run_device", "pch_run_rows", "pch_run_rows_device",
           "pch_fps", "pch_probe", "pch_half_edge_build", "pch_half_edge_error")

_lib = None


def load():
    """Load libpch_b200.so and declare its signatures (no GPU needed)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeUnavailable(
            f"{LIB_PATH} is not built; run paper_1305_1293_b200.build.build_native()")
    lib = ctypes.CDLL(LIB_PATH)
    P = ctypes.c_void_p
    i64 = ctypes.c_int64
    lib.pch_abi_version.restype = ctypes.c_int
    lib.pch_last_error.restype = ctypes.c_char_p
    lib.pch_device_count.restype = ctypes.c_int
    lib.pch_mesh_create.argtypes = [P, P, P, P, P, P, i64, i64, ctypes.c_int32,
                                    ctypes.POINTER(ctypes.c_void_p)]
    lib.pch_mesh_create.restype = ctypes.c_int
    lib.pch_mesh_destroy.argtypes = [P]
    lib.pch_mesh_destroy.restype = ctypes.c_int
    lib.pch_mesh_device_bytes.argtypes = [P]
    lib.pch_mesh_device_bytes.restype = i64
    lib.pch_run.argtypes = [P, P, i64, ctypes.POINTER(PchConfig), P,
                            ctypes.POINTER(PchStats)]
    lib.pch_run.restype = ctypes.c_int
    lib.pch_run_device.argtypes = [P, P, i64, ctypes.POINTER(PchConfig), P, P,
                                   ctypes.POINTER(PchStats)]
    lib.pch_run_device.restype = ctypes.c_int
    lib.pch_run_rows.argtypes = [P, P, i64, ctypes.POINTER(PchConfig), P,
                                 ctypes.POINTER(PchStats)]
    lib.pch_run_rows.restype = ctypes.c_int
    lib.pch_run_rows_device.argtypes = [P, P, i64, ctypes.POINTER(PchConfig), P, P,
                                        ctypes.POINTER(PchStats)]
    lib.pch_run_rows_device.restype = ctypes.c_int
    lib.pch_fps.argtypes = [P, i64, i64, ctypes.POINTER(PchConfig), P, P,
                            ctypes.POINTER(PchStats)]
    lib.pch_fps.restype = ctypes.c_int
    lib.pch_probe.argtypes = [ctypes.c_int32, P, ctypes.c_int32]
    lib.pch_probe.restype = ctypes.c_int
    lib.pch_half_edge_build.argtypes = [P, i64, P, i64, P, P, P, P, P, P, P, P, ctypes.c_int32]
    lib.pch_half_edge_build.restype = ctypes.c_int
    lib.pch_half_edge_error.restype = ctypes.c_char_p
    if lib.pch_abi_version() != ABI_VERSION:
        raise NativeUnavailable("libpch_b200.so ABI version mismatch")
    _lib = lib
    return lib


def last_error() -> str:
    return load().pch_last_error().decode(errors="replace")
