"""ctypes wrapper for the CPU parity oracle (oracle/pch_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs, never by the product
package.  ``run_ich`` / ``run_pch`` restate the reference engines
(reference pkg/src/pargeo/engine.py:624 run_ich, :433 run_pch) and return
``(dist, stats_dict)``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "libpch_oracle.so")

STAT_FIELDS = ("iterations", "windows_propagated", "total_windows_created",
               "total_windows_pruned", "pruned_ich", "pruned_split",
               "pruned_tiny", "pruned_degenerate", "pruned_duplicate",
               "windows_stored", "max_children_per_window", "events_created",
               "events_applied", "peak_active_pool")


class _Stats(ctypes.Structure):
    _fields_ = [(f, ctypes.c_int64) for f in STAT_FIELDS]


_lib = None


def build() -> str:
    """Compile the oracle with its Makefile (gcc; no GPU needed)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        lib = ctypes.CDLL(_LIB_PATH)
        p = ctypes.c_void_p
        i64 = ctypes.c_int64
        lib.pch_oracle_run_ich.argtypes = [p, p, p, p, p, p, i64, i64, p, i64,
                                          ctypes.c_double, ctypes.c_int, p, p]
        lib.pch_oracle_run_pch.argtypes = [p, p, p, p, p, p, i64, i64, p, i64,
                                          i64, ctypes.c_int, ctypes.c_int,
                                          ctypes.c_double, ctypes.c_int, i64,
                                          p, p]
        lib.pch_oracle_run_ich.restype = ctypes.c_int
        lib.pch_oracle_run_pch.restype = ctypes.c_int
        _lib = lib
    return _lib


def _mesh_args(mesh):
    arrs = (np.ascontiguousarray(mesh.origin, np.int64),
            np.ascontiguousarray(mesh.opposite, np.int64),
            np.ascontiguousarray(mesh.length, np.float64),
            np.ascontiguousarray(mesh.corner_angle, np.float64),
            np.ascontiguousarray(mesh.vertex_class, np.uint8),
            np.ascontiguousarray(mesh.outgoing, np.int64))
    return arrs, [a.ctypes.data for a in arrs]


def _sources(mesh, sources):
    src = sorted(set(int(s) for s in sources))
    if not src:
        raise ValueError("at least one source vertex is required")
    for s in src:
        if s < 0 or s >= mesh.n_vertices:
            raise ValueError(f"invalid source index {s}")
    return np.asarray(src, np.int64)


def run_ich(mesh, sources, epsilon_window=1e-6, fan_mode="clip"):
    lib = _load()
    keep, ptrs = _mesh_args(mesh)
    src = _sources(mesh, sources)
    dist = np.empty(mesh.n_vertices)
    st = _Stats()
    rc = lib.pch_oracle_run_ich(*ptrs, mesh.n_vertices, mesh.n_faces,
                                src.ctypes.data, len(src), epsilon_window,
                                int(fan_mode == "full_edges"),
                                dist.ctypes.data, ctypes.byref(st))
    if rc:
        raise RuntimeError(f"oracle run_ich failed ({rc})")
    return dist, {f: int(getattr(st, f)) for f in STAT_FIELDS}


def run_pch(mesh, sources, k=4096, workers=1, selection_mode="exact",
            epsilon_window=1e-6, fan_mode="clip", max_iterations=None):
    lib = _load()
    keep, ptrs = _mesh_args(mesh)
    src = _sources(mesh, sources)
    dist = np.empty(mesh.n_vertices)
    st = _Stats()
    rc = lib.pch_oracle_run_pch(*ptrs, mesh.n_vertices, mesh.n_faces,
                                src.ctypes.data, len(src), int(k),
                                int(workers),
                                int(selection_mode == "approximate_strided"),
                                epsilon_window, int(fan_mode == "full_edges"),
                                int(max_iterations or 0),
                                dist.ctypes.data, ctypes.byref(st))
    if rc == -2:
        raise RuntimeError(f"iteration cap {max_iterations} exceeded")
    if rc:
        raise RuntimeError(f"oracle run_pch failed ({rc})")
    return dist, {f: int(getattr(st, f)) for f in STAT_FIELDS}
