"""B200-native Parallel Chen-Han (PCH) exact geodesic distance solver.

Drop-in for the hot path of the reference package ``pargeo``
(``run_pch(mesh, sources, config) -> (dist, stats)``): mesh arrays and
source indices in, per-vertex exact geodesic distances out, computed by a
persistent sm_100a kernel behind the C ABI in ``include/pch_b200.h``.
"""
from .engine import (DeviceMesh, EngineConfig, EngineGuard, RunStats,
                     device_mesh, farthest_point_sampling, run_pch,
                     run_pch_device, run_pch_rows, run_pch_rows_device)
from .mesh import (BOUNDARY, MeshError, SurfaceMesh, VertexClass,
                   build_half_edge_mesh, classify_total_angle,
                   next_half_edge, prev_half_edge)

__version__ = "0.1.0"

__all__ = [
    "BOUNDARY", "DeviceMesh", "EngineConfig", "EngineGuard", "MeshError",
    "RunStats", "SurfaceMesh", "VertexClass", "build_half_edge_mesh",
    "classify_total_angle", "device_mesh", "farthest_point_sampling",
    "next_half_edge",
    "prev_half_edge", "run_pch", "run_pch_device", "run_pch_rows",
    "run_pch_rows_device",
]
