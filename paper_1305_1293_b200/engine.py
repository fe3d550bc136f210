"""Engine entry points -- the drop-in for the reference's ``pargeo.engine``
hot path.

``run_pch(mesh, sources, config) -> (dist, RunStats)`` keeps the
reference signature, argument meaning and error behaviour (reference
pkg/src/pargeo/engine.py:433; ``EngineConfig`` :44, ``RunStats`` :76,
``EngineGuard`` :40, source validation :392).  The work happens in the
CUDA library behind the C ABI (include/pch_b200.h): the mesh is uploaded
once per (mesh, device) and stays resident; each call ships only the
source indices in and the distance field out.

There is deliberately no CPU path here: without the library or a CUDA
device every call raises.
"""
from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass, fields

import numpy as np

from . import _native
from .mesh import SurfaceMesh

SELECTION_MODES = ("exact", "approximate_strided")
FAN_MODES = ("clip", "full_edges")
TINY_RULES = ("angular", "absolute")


class EngineGuard(RuntimeError):
    """A configured safety guard stopped the run (engine.py:40)."""


@dataclass
class EngineConfig:
    """Engine parameters (engine.py:44).

    ``k`` is the per-iteration selection size: the device steers the
    distance threshold so that about ``k`` windows fall below it and
    propagates all of them.  The default is the paper's GPU optimum
    (§5.2: k in [16, 24] x 2^10 on 512-core GPUs); the reference's 4096 is
    its CPU-worker setting.  ``workers`` is accepted for
    interface parity; on the device every selected window gets its own
    thread.  ``selection_mode`` applies to the two-barrier (deterministic)
    solver's k-selection: "exact" refines the histogram bin holding the
    k-th key into 1024 sub-bins (the k nearest windows, reference
    argpartition, engine.py:256), "approximate_strided" takes the whole
    bin; the default one-barrier solver steers a distance step by k
    instead (results are identical for any selection, paper §4.3).  ``recheck`` enables the pop-time endpoint
    re-check of the ICH filter; ``pool_capacity`` is the initial window
    pool size (0 = automatic; the pool doubles on overflow).
    ``deterministic`` selects the two-barrier solver whose filters read
    tables frozen at the start of each iteration (the paper's delayed
    update): fields are then bitwise identical across runs.  The default
    one-barrier solver reads the live tables and is faster; its fields
    agree across runs to rounding (far inside the 1e-9 bar).
    ``chain`` bounds how many propagations one thread performs per
    iteration when a child falls inside the next batch's threshold (it is
    then propagated at once instead of waiting for the next iteration);
    0 = library default (3 on meshes of >= 2^18 faces, 6 if their faces
    are anisotropic, else 2), 1 = off.
    ``max_iterations`` has the reference's meaning (None: no cap; n: raise
    ``EngineGuard`` once more than n iterations ran, engine.py:475);
    ``time_limit_s`` is an optional device wall-time guard (0 = none; no
    reference counterpart), also raising ``EngineGuard``.
    ``tiny_rule`` selects the tiny-window drop: "absolute" is the
    reference's (width <= epsilon_window, geom.py:133); the default
    "angular" scales the threshold with the distance to the pseudo source
    within 40 mean edges, so the thin fans of nearly flat saddles survive
    (the reference's rounding holes behind such saddles).
    ``fan_margin`` widens every saddle fan by that angle (radians) on both
    sides; 0 is the reference's clip.  With ``deterministic=True`` a margin
    of 1e-5 removes the remaining rounding slivers on the 4M-face torus
    knot.  ``phase_times`` fills RunStats.time_select /
    _propagate / _compact / _events (the four phases run fused in one
    kernel; the device attributes its warp cycles to them, ~3 % slower).
    ``dedupe`` drops exact-duplicate fan windows as the reference does
    (engine.py:201, counted in RunStats.pruned_duplicate); off by default
    (the per-vertex fan pick leaves ~0.02 % twins; the table costs ~10 %).
    """

    k: int = 16384
    workers: int = 1
    selection_mode: str = "exact"
    epsilon_window: float = 1e-6
    seed: int = 0
    max_iterations: int | None = None
    fan_mode: str = "clip"
    device: int = 0
    recheck: bool = True
    pool_capacity: int = 0
    deterministic: bool = False
    chain: int = 0
    time_limit_s: float = 0.0
    tiny_rule: str = "angular"
    fan_margin: float = 0.0
    phase_times: bool = False
    dedupe: bool = False

    def __post_init__(self):
        if self.k < 1:
            raise ValueError("k must be >= 1")
        if self.workers < 1:
            raise ValueError("workers must be >= 1")
        if self.selection_mode not in SELECTION_MODES:
            raise ValueError(f"selection_mode must be one of {SELECTION_MODES}")
        if self.fan_mode not in FAN_MODES:
            raise ValueError(f"fan_mode must be one of {FAN_MODES}")
        if not self.epsilon_window > 0.0:
            raise ValueError("epsilon_window must be > 0")
        if self.chain < 0:
            raise ValueError("chain must be >= 0")
        if self.time_limit_s < 0:
            raise ValueError("time_limit_s must be >= 0")
        if not 0.0 <= self.fan_margin < 0.1:
            raise ValueError("fan_margin must be in [0, 0.1)")
        if self.tiny_rule not in TINY_RULES:
            raise ValueError(f"tiny_rule must be one of {TINY_RULES}")

    def to_native(self) -> _native.PchConfig:
        c = _native.PchConfig()
        c.k = int(self.k)
        c.selection_mode = SELECTION_MODES.index(self.selection_mode)
        c.fan_mode = FAN_MODES.index(self.fan_mode)
        c.epsilon_window = float(self.epsilon_window)
        c.max_iterations = -1 if self.max_iterations is None else int(self.max_iterations)
        c.pool_capacity = int(self.pool_capacity)
        c.flags = ((0 if self.recheck else _native.FLAG_NO_RECHECK)
                   | (_native.FLAG_DETERMINISTIC if self.deterministic else 0)
                   | (_native.FLAG_ABSOLUTE_TINY if self.tiny_rule == "absolute" else 0)
                   | (_native.FLAG_PHASE_TIMES if self.phase_times else 0)
                   | (_native.FLAG_DEDUPE if self.dedupe else 0))
        c.chain = int(self.chain)
        c.time_limit_s = float(self.time_limit_s)
        c.fan_margin = float(self.fan_margin)
        return c


@dataclass
class RunStats:
    """Run accounting (engine.py:76) plus device counters."""

    algorithm: str = ""
    iterations: int = 0
    windows_propagated: int = 0
    total_windows_created: int = 0
    total_windows_pruned: int = 0
    pruned_ich: int = 0
    pruned_split: int = 0
    pruned_tiny: int = 0
    pruned_degenerate: int = 0
    pruned_duplicate: int = 0
    pruned_recheck: int = 0
    windows_stored: int = 0
    max_children_per_window: int = 0
    events_created: int = 0
    events_applied: int = 0
    peak_active_pool: int = 0
    fans_emitted: int = 0
    buffer_regrows: int = 0
    pool_restarts: int = 0
    grid_barriers: int = 0
    time_total: float = 0.0
    time_select: float = 0.0
    time_propagate: float = 0.0
    time_compact: float = 0.0
    time_events: float = 0.0
    time_device_ms: float = 0.0
    time_kernel_ms: float = 0.0
    prop_item_us: float = 0.0

    def to_dict(self) -> dict:
        return {f.name: getattr(self, f.name) for f in fields(self)}

    @classmethod
    def from_native(cls, st: _native.PchStats, algorithm="pch-b200"):
        s = cls(algorithm=algorithm)
        for f in _native.STAT_FIELDS:
            setattr(s, f, int(getattr(st, f)))
        s.time_device_ms = float(st.time_total_ms)
        s.time_kernel_ms = float(st.time_kernel_ms)
        s.time_total = s.time_device_ms / 1e3
        # the four phases are fused into one kernel: the device attributes
        # its warp cycles to them (include/pch_b200.h pch_stats)
        s.time_select = float(st.time_select_ms) / 1e3
        s.time_propagate = float(st.time_propagate_ms) / 1e3
        s.time_compact = float(st.time_compact_ms) / 1e3
        s.time_events = float(st.time_events_ms) / 1e3
        s.prop_item_us = float(st.prop_item_us)
        return s


class DeviceMesh:
    """A mesh resident on one GPU (the paper's §4.1 tables plus
    precomputed per-half-edge unfoldings and per-vertex fan wedges)."""

    def __init__(self, mesh: SurfaceMesh, device: int = 0):
        lib = _native.load()
        if lib.pch_device_count() <= device:
            raise _native.NativeUnavailable(
                f"no CUDA device {device} visible to libpch_b200")
        arrs = (np.ascontiguousarray(mesh.origin, np.int64),
                np.ascontiguousarray(mesh.opposite, np.int64),
                np.ascontiguousarray(mesh.length, np.float64),
                np.ascontiguousarray(mesh.corner_angle, np.float64),
                np.ascontiguousarray(mesh.vertex_class, np.uint8),
                np.ascontiguousarray(mesh.outgoing, np.int64))
        handle = ctypes.c_void_p()
        rc = lib.pch_mesh_create(*[a.ctypes.data for a in arrs],
                                 mesh.n_vertices, mesh.n_faces, int(device),
                                 ctypes.byref(handle))
        _check(rc)
        self.handle = handle
        self.device = device
        self.n_vertices = mesh.n_vertices
        self._lib = lib
        # one solve at a time per device mesh: the native workspace (window
        # pools, tables, stream) belongs to the mesh handle, and ctypes
        # releases the GIL during the call
        self.lock = threading.Lock()

    @property
    def device_bytes(self) -> int:
        return int(self._lib.pch_mesh_device_bytes(self.handle))

    def close(self):
        if self.handle:
            self._lib.pch_mesh_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _check(rc: int):
    if rc == _native.PCH_OK:
        return
    msg = _native.last_error()
    if rc in (_native.PCH_ERR_SOURCE, _native.PCH_ERR_CONFIG, _native.PCH_ERR_MESH):
        raise ValueError(msg)
    if rc == _native.PCH_ERR_GUARD:
        raise EngineGuard(msg)
    raise RuntimeError(f"libpch_b200 error {rc}: {msg}")


def device_mesh(mesh: SurfaceMesh, device: int = 0) -> DeviceMesh:
    """The cached device-resident copy of ``mesh`` on ``device``."""
    cache = mesh.__dict__.setdefault("_pch_device_meshes", {})
    dm = cache.get(device)
    if dm is None or dm.handle is None:
        dm = DeviceMesh(mesh, device)
        cache[device] = dm
    return dm


def _check_sources(mesh: SurfaceMesh, sources) -> np.ndarray:
    """engine.py:392 -- non-empty, in range, deduplicated and sorted."""
    src = [int(s) for s in sources]
    if not src:
        raise ValueError("at least one source vertex is required")
    for s in src:
        if s < 0 or s >= mesh.n_vertices:
            raise ValueError(f"invalid source index {s}")
    return np.asarray(sorted(set(src)), dtype=np.int64)


_PINNED_MAX_BYTES = 1 << 28


def _host_field(n: int) -> np.ndarray:
    """A float64 host array for a field read back from the device: in
    page-locked memory (torch's caching host allocator -- the device copy
    runs at full link speed, 4 MB: 0.09 ms instead of 0.27 ms pageable;
    views keep the block alive like any numpy array), or plain numpy
    memory when that is unavailable or the array is large."""
    if 8 * n <= _PINNED_MAX_BYTES:
        try:
            import torch
            if torch.cuda.is_available():
                return torch.empty(n, dtype=torch.float64, pin_memory=True).numpy()
        except Exception:  # allocation plumbing only; the solve is native either way
            pass
    return np.empty(n, dtype=np.float64)


def run_pch(mesh: SurfaceMesh, sources, config: EngineConfig | None = None):
    """Exact geodesic distances from the source vertices on the GPU.

    Returns ``(distance_field, RunStats)``; +inf marks vertices no window
    reaches (boundary shadows), exactly as the reference does."""
    config = config or EngineConfig()
    src = _check_sources(mesh, sources)
    dm = device_mesh(mesh, config.device)
    out = _host_field(mesh.n_vertices)
    st = _native.PchStats()
    cfg = config.to_native()
    with dm.lock:
        rc = dm._lib.pch_run(dm.handle, src.ctypes.data, len(src),
                             ctypes.byref(cfg), out.ctypes.data, ctypes.byref(st))
    _check(rc)
    return out, RunStats.from_native(st)


def run_pch_rows(mesh: SurfaceMesh, sources, config: EngineConfig | None = None):
    """One single-source field per source (distance-matrix rows): returns
    ``(rows[len(sources), n_vertices], RunStats)``; sources keep their
    order and duplicates."""
    config = config or EngineConfig()
    src = np.asarray([int(s) for s in sources], dtype=np.int64)
    if len(src) == 0:
        raise ValueError("at least one source vertex is required")
    if src.min() < 0 or src.max() >= mesh.n_vertices:
        bad = int(src[(src < 0) | (src >= mesh.n_vertices)][0])
        raise ValueError(f"invalid source index {bad}")
    dm = device_mesh(mesh, config.device)
    out = np.empty((len(src), mesh.n_vertices), dtype=np.float64)
    st = _native.PchStats()
    cfg = config.to_native()
    with dm.lock:
        rc = dm._lib.pch_run_rows(dm.handle, src.ctypes.data, len(src),
                                  ctypes.byref(cfg), out.ctypes.data,
                                  ctypes.byref(st))
    _check(rc)
    return out, RunStats.from_native(st)


def farthest_point_sampling(mesh: SurfaceMesh, n_samples: int, first: int = 0,
                            config: EngineConfig | None = None):
    """Greedy geodesic farthest-point sampling: sample 0 is ``first``,
    sample s+1 the vertex farthest from samples 0..s (ties: lowest index;
    unreached components first).  Returns ``(samples int64[n_samples],
    min_field float64[n_vertices], RunStats)`` where ``min_field`` equals
    ``run_pch(mesh, samples)[0]``.  One seeded solve per sample on the
    device (include/pch_b200.h: pch_fps)."""
    config = config or EngineConfig()
    n = int(n_samples)
    if n < 1:
        raise ValueError("n_samples must be >= 1")
    first = int(first)
    if first < 0 or first >= mesh.n_vertices:
        raise ValueError(f"invalid source index {first}")
    dm = device_mesh(mesh, config.device)
    samples = np.empty(n, dtype=np.int64)
    out = _host_field(mesh.n_vertices)
    st = _native.PchStats()
    cfg = config.to_native()
    with dm.lock:
        rc = dm._lib.pch_fps(dm.handle, first, n, ctypes.byref(cfg), samples.ctypes.data,
                             out.ctypes.data, ctypes.byref(st))
    _check(rc)
    return samples, out, RunStats.from_native(st)


def run_pch_device(mesh: SurfaceMesh, d_sources_ptr: int, n_sources: int,
                   d_out_ptr: int, config: EngineConfig | None = None,
                   stream: int = 0):
    """Device-pointer variant (inputs already resident in HBM): sources
    int64[n] and output float64[n_vertices] on the mesh's device."""
    config = config or EngineConfig()
    dm = device_mesh(mesh, config.device)
    st = _native.PchStats()
    cfg = config.to_native()
    with dm.lock:
        rc = dm._lib.pch_run_device(dm.handle, ctypes.c_void_p(d_sources_ptr),
                                    int(n_sources), ctypes.byref(cfg),
                                    ctypes.c_void_p(d_out_ptr),
                                    ctypes.c_void_p(stream or None),
                                    ctypes.byref(st))
    _check(rc)
    return RunStats.from_native(st)


def run_pch_rows_device(mesh: SurfaceMesh, d_sources_ptr: int, n_sources: int,
                        d_out_ptr: int, config: EngineConfig | None = None,
                        stream: int = 0):
    """Device-pointer rows (include/pch_b200.h pch_run_rows_device): sources
    int64[n] and output float64[n, n_vertices] resident on the mesh's
    device; the rows never cross PCIe (shard.py gathers them over NCCL)."""
    config = config or EngineConfig()
    dm = device_mesh(mesh, config.device)
    st = _native.PchStats()
    cfg = config.to_native()
    with dm.lock:
        rc = dm._lib.pch_run_rows_device(dm.handle, ctypes.c_void_p(d_sources_ptr),
                                         int(n_sources), ctypes.byref(cfg),
                                         ctypes.c_void_p(d_out_ptr),
                                         ctypes.c_void_p(stream or None),
                                         ctypes.byref(st))
    _check(rc)
    return RunStats.from_native(st)


def probe(device: int = 0) -> dict:
    """Roofline denominators measured on the device (include/pch_b200.h
    pch_probe): FP64 FMA TFLOP/s and the live solver's grid-barrier us."""
    lib = _native.load()
    out = (ctypes.c_double * 2)()
    _check(lib.pch_probe(int(device), out, 2))
    return {"fp64_tflops": float(out[0]), "grid_barrier_us": float(out[1])}
