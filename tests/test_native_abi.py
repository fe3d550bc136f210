"""The C ABI boundary: the shared library loads (no GPU needed), exports
every symbol include/pch_b200.h declares, and the Python layer mirrors the
reference's argument validation before any device work."""
import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT
from paper_1305_1293_b200 import EngineConfig, RunStats, _native, meshes
from paper_1305_1293_b200.engine import _check_sources

HEADER = os.path.join(ROOT, "include", "pch_b200.h")


def _declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(pch_[a-z_0-9]+)\s*\(",
                                 text, re.M)))


def test_header_declares_entry_points():
    syms = _declared_symbols()
    assert {"pch_mesh_create", "pch_run", "pch_run_device", "pch_run_rows"} <= set(syms)
    assert sorted(_native.EXPORTS) == syms


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_native.LIB_PATH)
    for s in _declared_symbols():
        assert hasattr(lib, s), s


def test_library_loads_and_reports_abi():
    lib = _native.load()
    assert lib.pch_abi_version() == _native.ABI_VERSION
    assert lib.pch_device_count() >= 0


def test_struct_layouts_match_header():
    # pch_config: 8+4+4+8+8+8+4+4+8+8 ; pch_stats: 19 int64 + 7 doubles
    assert ctypes.sizeof(_native.PchConfig) == 64
    assert ctypes.sizeof(_native.PchStats) == 8 * 26


def test_sass_is_sm100a():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", _native.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_engine_config_validation():
    with pytest.raises(ValueError):
        EngineConfig(k=0)
    with pytest.raises(ValueError):
        EngineConfig(workers=0)
    with pytest.raises(ValueError):
        EngineConfig(selection_mode="sorted")
    with pytest.raises(ValueError):
        EngineConfig(fan_mode="none")
    with pytest.raises(ValueError):
        EngineConfig(chain=-1)
    c = EngineConfig(k=123, fan_mode="full_edges", recheck=False, chain=3).to_native()
    assert (c.k, c.fan_mode, c.flags, c.chain) == (123, 1, _native.FLAG_NO_RECHECK, 3)
    c = EngineConfig(deterministic=True).to_native()
    assert c.flags == _native.FLAG_DETERMINISTIC
    with pytest.raises(ValueError):
        EngineConfig(time_limit_s=-1.0)
    # reference semantics (engine.py:475): None = no cap, 0 = a real cap
    assert EngineConfig().to_native().max_iterations == -1
    assert EngineConfig(max_iterations=0).to_native().max_iterations == 0
    assert EngineConfig(time_limit_s=2.5).to_native().time_limit_s == 2.5


def test_source_validation_matches_reference(cube):
    with pytest.raises(ValueError):
        _check_sources(cube, [])
    with pytest.raises(ValueError, match="invalid source index 99"):
        _check_sources(cube, [99])
    with pytest.raises(ValueError):
        _check_sources(cube, [-1])
    assert _check_sources(cube, [3, 1, 3]).tolist() == [1, 3]


def test_runstats_to_dict_flat():
    s = RunStats(algorithm="pch-b200", iterations=3)
    d = s.to_dict()
    assert d["algorithm"] == "pch-b200" and d["iterations"] == 3
    assert all(isinstance(v, (int, float, str)) for v in d.values())


def test_no_device_raises_loudly():
    """On a machine without a GPU the product path must fail, not fall
    back to a CPU implementation."""
    lib = _native.load()
    if lib.pch_device_count() > 0:
        pytest.skip("a CUDA device is present")
    from paper_1305_1293_b200 import run_pch
    with pytest.raises(_native.NativeUnavailable):
        run_pch(meshes.make("cube"), [0])


def test_fps_argument_validation(cube):
    """farthest_point_sampling rejects bad arguments before touching the
    device (the same ValueError contract as run_pch's sources)."""
    from paper_1305_1293_b200 import farthest_point_sampling
    with pytest.raises(ValueError):
        farthest_point_sampling(cube, 0, 0)
    with pytest.raises(ValueError, match="invalid source index"):
        farthest_point_sampling(cube, 2, cube.n_vertices)
    with pytest.raises(ValueError):
        farthest_point_sampling(cube, 2, -1)


def test_fps_no_device_raises_loudly(cube):
    lib = _native.load()
    if lib.pch_device_count() > 0:
        pytest.skip("a CUDA device is present")
    from paper_1305_1293_b200 import farthest_point_sampling
    with pytest.raises(_native.NativeUnavailable):
        farthest_point_sampling(cube, 2, 0)


def test_host_field_is_plain_numpy_without_cuda():
    """Without a visible GPU the readback buffer is ordinary numpy memory
    (the page-locked allocator is only plumbing for the device copy)."""
    from paper_1305_1293_b200.engine import _host_field
    a = _host_field(1000)
    assert a.shape == (1000,) and a.dtype == np.float64 and a.flags.writeable
