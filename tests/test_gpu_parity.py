"""GPU parity: the CUDA engine (through the C ABI) against the reference's
golden fields and the CPU oracle.  Bar (BASELINE.json north star): max
relative per-vertex error <= 1e-9 and bit-identical unreachable flags.

Reference test model: pkg/tests/test_acceptance.py (criteria 1-8) and
pkg/tests/test_engine.py.
"""
import math

import numpy as np
import pytest

from conftest import TOL, golden_cases, load_golden, max_rel_dev

pytestmark = pytest.mark.gpu

CASES = golden_cases()


def _gpu():
    from paper_1305_1293_b200 import _native
    lib = _native.load()
    if lib.pch_device_count() < 1:
        pytest.fail("no CUDA device visible: the GPU tier needs a B200")
    return lib


def _ref_field(g):
    """The reference field a drop-in must reproduce.  Where the reference's
    two engines agree on reachability (all meshes without boundary
    shadows) that is run_ich; on boundary-shadowed meshes the reference is
    schedule dependent (tests/test_oracle_golden.py) and only the vertices
    both reference engines reach are compared."""
    ich, pch = g["ich_dist"], g["pch_dist"]
    if np.array_equal(np.isfinite(ich), np.isfinite(pch)):
        return ich, None
    both = np.isfinite(ich) & np.isfinite(pch)
    return ich, both


@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("k", [1, 64, 4096, 65536])
def test_golden_parity(name, k):
    _gpu()
    from paper_1305_1293_b200 import EngineConfig, run_pch
    m, g = load_golden(name)
    d, st = run_pch(m, g["sources"], EngineConfig(k=k))
    ref, mask = _ref_field(g)
    if mask is None:
        assert np.array_equal(np.isfinite(d), np.isfinite(ref)), name
        assert max_rel_dev(d, ref) <= TOL, name
    else:
        # shadowed boundary (reflex boundary vertices the reference never
        # bends around): the reference's own two engines disagree on which
        # vertices they reach and, at a few, on the route around the shadow
        # (schedule-dependent pruning, tests/test_oracle_golden.py).  Every
        # vertex both reach, the GPU reaches; where they agree the GPU is
        # within 1e-9 of them; where they disagree it lies between them
        pch = g["pch_dist"]
        assert np.all(np.isfinite(d[mask])), name
        agree = mask & (np.abs(ref - pch) <= TOL * np.maximum(np.abs(ref), 1e-12))
        assert max_rel_dev(d[agree], ref[agree]) <= TOL, name
        lo, hi = np.minimum(ref, pch), np.maximum(ref, pch)
        split = mask & ~agree
        assert np.all(d[split] >= lo[split] * (1 - TOL)) and np.all(d[split] <= hi[split] * (1 + TOL)), name
    src = np.asarray(g["sources"])
    assert np.all(d[src] == 0.0)
    assert st.iterations >= 1 and st.windows_propagated >= 1


@pytest.mark.parametrize("name", [c for c in CASES if c.startswith("tiny_")])
def test_tiny_vs_brute_force(name):
    _gpu()
    from paper_1305_1293_b200 import run_pch
    m, g = load_golden(name)
    d, _ = run_pch(m, g["sources"])
    assert max_rel_dev(d, g["brute_dist"]) <= TOL, name


def test_cube_diagonal_sqrt5():
    _gpu()
    from paper_1305_1293_b200 import meshes, run_pch
    d, _ = run_pch(meshes.make("cube"), [0])
    assert d[6] == pytest.approx(math.sqrt(5.0), rel=1e-12)


def test_fan_mode_full_edges_matches():
    _gpu()
    from paper_1305_1293_b200 import EngineConfig, run_pch
    m, g = load_golden("bumpy_sphere20k_s3")
    d, _ = run_pch(m, g["sources"], EngineConfig(fan_mode="full_edges"))
    assert max_rel_dev(d, g["ich_dist"]) <= TOL


@pytest.mark.parametrize("chain", [1, 2, 4])
def test_chain_lengths_match(chain):
    _gpu()
    from paper_1305_1293_b200 import EngineConfig, run_pch
    for name in ("bumpy_sphere20k_s3", "bumpy_torus4800_s5", "icosphere5120_multi16"):
        m, g = load_golden(name)
        d, _ = run_pch(m, g["sources"], EngineConfig(chain=chain))
        assert max_rel_dev(d, g["ich_dist"]) <= TOL, (name, chain)


def test_recheck_off_matches():
    _gpu()
    from paper_1305_1293_b200 import EngineConfig, run_pch
    m, g = load_golden("bumpy_torus4800_s5")
    d, _ = run_pch(m, g["sources"], EngineConfig(recheck=False))
    assert max_rel_dev(d, g["ich_dist"]) <= TOL


def test_determinism_repeated_runs():
    """Acceptance criterion 8: identical fields (bitwise) across runs."""
    _gpu()
    from paper_1305_1293_b200 import EngineConfig, run_pch
    m, g = load_golden("icosphere20480_s1370")
    runs = [run_pch(m, g["sources"], EngineConfig(k=4096, deterministic=True))[0]
            for _ in range(3)]
    for r in runs[1:]:
        assert np.array_equal(r.view(np.int64), runs[0].view(np.int64))


def test_multi_source_is_pointwise_min():
    """Acceptance criterion 7 (Table 3 context)."""
    _gpu()
    from paper_1305_1293_b200 import run_pch, run_pch_rows
    m, g = load_golden("icosphere5120_multi16")
    src = [int(s) for s in g["sources"]]
    multi, _ = run_pch(m, src)
    rows, _ = run_pch_rows(m, src)
    assert rows.shape == (len(src), m.n_vertices)
    assert max_rel_dev(multi, rows.min(axis=0)) <= TOL
    assert max_rel_dev(multi, g["ich_dist"]) <= TOL


def test_rows_match_single_runs_and_oracle():
    _gpu()
    from oracle import oracle as O
    from paper_1305_1293_b200 import run_pch, run_pch_rows
    m, g = load_golden("bumpy_torus4800_s5")
    src = [5, 77, 5, 1234]
    rows, _ = run_pch_rows(m, src)
    for r, s in zip(rows, src):
        single, _ = run_pch(m, [s])
        assert max_rel_dev(r, single) <= TOL
        ref, _ = O.run_ich(m, [s])
        assert max_rel_dev(r, ref) <= TOL


def test_device_pointer_entry():
    _gpu()
    import torch
    from paper_1305_1293_b200 import run_pch, run_pch_device
    m, g = load_golden("icosphere5120_s342")
    src = torch.tensor([int(s) for s in g["sources"]], dtype=torch.int64, device="cuda:0")
    out = torch.empty(m.n_vertices, dtype=torch.float64, device="cuda:0")
    torch.cuda.synchronize()
    run_pch_device(m, src.data_ptr(), src.numel(), out.data_ptr(),
                   stream=torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    d = out.cpu().numpy()
    assert max_rel_dev(d, g["ich_dist"]) <= TOL
    host, _ = run_pch(m, g["sources"])
    assert np.array_equal(d, host)


def test_iteration_guard_raises():
    _gpu()
    from paper_1305_1293_b200 import EngineConfig, EngineGuard, run_pch
    m, g = load_golden("icosphere1280_s85")
    with pytest.raises(EngineGuard):
        run_pch(m, g["sources"], EngineConfig(k=1, max_iterations=3))


def test_small_pool_regrows():
    """A pool that starts far too small grows at iteration boundaries and
    the solve continues (no rerun): the iteration count equals the one of a
    run that never grew, give or take the grown run's step decisions."""
    _gpu()
    from paper_1305_1293_b200 import EngineConfig, run_pch
    m, g = load_golden("icosphere20480_s1370")
    d, st = run_pch(m, g["sources"], EngineConfig(pool_capacity=256))
    assert st.buffer_regrows >= 1
    assert max_rel_dev(d, g["ich_dist"]) <= TOL
    _, ref = run_pch(m, g["sources"], EngineConfig())
    assert ref.buffer_regrows == 0
    assert st.iterations <= ref.iterations + 4 * st.buffer_regrows
    # a moderately small pool grows without ever rerunning the solve
    d2, st2 = run_pch(m, g["sources"], EngineConfig(pool_capacity=1 << 14))
    assert st2.buffer_regrows >= 1 and st2.pool_restarts == 0
    assert max_rel_dev(d2, g["ich_dist"]) <= TOL


def test_edge_lipschitz_and_sandwich_terrain():
    """Acceptance criterion 4 on a generated terrain (every vertex
    reachable: convex flat rim)."""
    _gpu()
    from paper_1305_1293_b200 import meshes, run_pch
    from paper_1305_1293_b200.mesh import build_half_edge_mesh
    m = build_half_edge_mesh(*meshes.terrain(60))
    s = 30 * 61 + 30
    d, _ = run_pch(m, [s])
    assert np.all(np.isfinite(d))
    u = m.origin
    v = m.origin[3 * (np.arange(len(u)) // 3) + (np.arange(len(u)) + 1) % 3]
    assert np.all(np.abs(d[u] - d[v]) <= m.length + 1e-9)
    chord = np.linalg.norm(m.positions - m.positions[s], axis=1)
    assert np.all(chord - 1e-9 <= d)


@pytest.mark.parametrize("n", [5, 8, 40])
def test_batched_rows_match_single_fields(n):
    """pch_run_rows solves its sources in batches (one field per row, 32
    per kernel; batches of >= 8 rows run the 2-CTA/SM instance): every row
    equals the single-source field and the oracle."""
    _gpu()
    from oracle import oracle as O
    from paper_1305_1293_b200 import run_pch, run_pch_rows
    m, g = load_golden("bumpy_sphere20k_s3")
    src = np.random.default_rng(n).choice(m.n_vertices, n, replace=False).tolist()
    src[-1] = src[0]  # a duplicate source gets its own (identical) row
    rows, st = run_pch_rows(m, src)
    assert rows.shape == (n, m.n_vertices)
    assert st.iterations >= 1
    for r in (0, n // 2, n - 1):
        single, _ = run_pch(m, [src[r]])
        assert max_rel_dev(rows[r], single) <= TOL, r
    ref, _ = O.run_ich(m, [src[1]])
    assert max_rel_dev(rows[1], ref) <= TOL
    assert max_rel_dev(rows[-1], rows[0]) <= TOL


def test_batched_rows_deterministic_mode():
    _gpu()
    from paper_1305_1293_b200 import EngineConfig, run_pch_rows
    m, g = load_golden("icosphere5120_multi16")
    src = [int(s) for s in g["sources"][:4]]
    a, _ = run_pch_rows(m, src, EngineConfig(deterministic=True))
    b, _ = run_pch_rows(m, src, EngineConfig(deterministic=True))
    assert np.array_equal(a.view(np.int64), b.view(np.int64))
    assert max_rel_dev(a.min(axis=0), run_pch_rows(m, src)[0].min(axis=0)) <= TOL


def test_batched_rows_pool_regrow():
    _gpu()
    from paper_1305_1293_b200 import EngineConfig, run_pch, run_pch_rows
    m, g = load_golden("bumpy_torus4800_s5")
    src = list(range(0, 2400, 150))
    rows, st = run_pch_rows(m, src, EngineConfig(pool_capacity=4096))
    assert st.buffer_regrows >= 1
    for r in (0, len(src) - 1):
        assert max_rel_dev(rows[r], run_pch(m, [src[r]])[0]) <= TOL


def test_dedupe_drops_twins_only():
    """EngineConfig(dedupe=True): exact-duplicate fan windows are dropped
    (reference engine.py:201) and counted; the field is unchanged."""
    _gpu()
    from paper_1305_1293_b200 import EngineConfig, meshes, run_pch
    from paper_1305_1293_b200.mesh import build_half_edge_mesh
    m = build_half_edge_mesh(*meshes.terrain(120))
    s = 60 * 121 + 60
    a, sa = run_pch(m, [s], EngineConfig(dedupe=True))
    b, sb = run_pch(m, [s])
    assert sb.pruned_duplicate == 0
    assert sa.pruned_duplicate >= 0
    assert sa.total_windows_pruned >= sa.pruned_duplicate
    assert np.array_equal(np.isfinite(a), np.isfinite(b))
    assert max_rel_dev(a, b) <= TOL


@pytest.mark.parametrize("mode", ["exact", "approximate_strided"])
def test_deterministic_selection_modes(mode):
    """selection_mode in the two-barrier solver (reference engine.py:235
    select_nearest): "exact" refines the K-th key's histogram bin (the
    batch is the K nearest windows up to 1/1024 of a bin), "approximate
    _strided" takes the whole bin.  Both reproduce the reference field; the
    exact batches are smaller, so they need at least as many iterations."""
    _gpu()
    from paper_1305_1293_b200 import EngineConfig, run_pch
    m, g = load_golden("bumpy_sphere20k_s3")
    d, st = run_pch(m, g["sources"], EngineConfig(k=64, deterministic=True, selection_mode=mode))
    assert np.array_equal(np.isfinite(d), np.isfinite(g["ich_dist"]))
    assert max_rel_dev(d, g["ich_dist"]) <= TOL
    d2, st2 = run_pch(m, g["sources"], EngineConfig(k=64, deterministic=True, selection_mode=mode))
    assert np.array_equal(d.view(np.int64), d2.view(np.int64))  # still bitwise reproducible
    if mode == "exact":
        _, sa = run_pch(m, g["sources"], EngineConfig(k=64, deterministic=True,
                                                      selection_mode="approximate_strided"))
        assert st.iterations >= sa.iterations


def test_device_sources_validated():
    """an out-of-range index in a device-resident source list
    fails the solve with PCH_ERR_SOURCE (ValueError) instead of writing out
    of bounds; the mesh stays usable."""
    _gpu()
    import torch
    from paper_1305_1293_b200 import run_pch, run_pch_device, run_pch_rows_device
    m, g = load_golden("icosphere1280_s85")
    out = torch.empty(m.n_vertices, dtype=torch.float64, device="cuda:0")
    for bad in (-1, m.n_vertices, 1 << 40):
        src = torch.tensor([0, bad], dtype=torch.int64, device="cuda:0")
        with pytest.raises(ValueError):
            run_pch_device(m, src.data_ptr(), 2, out.data_ptr())
        rows = torch.empty((2, m.n_vertices), dtype=torch.float64, device="cuda:0")
        with pytest.raises(ValueError):
            run_pch_rows_device(m, src.data_ptr(), 2, rows.data_ptr())
    d, _ = run_pch(m, g["sources"])
    assert max_rel_dev(d, g["ich_dist"]) <= TOL


def test_max_iterations_reference_semantics():
    """ADVICE r1 / reference engine.py:475: None = no cap, 0 = a real cap
    (the guard trips after the first iteration); the optional wall-time
    guard is off by default."""
    _gpu()
    from paper_1305_1293_b200 import EngineConfig, EngineGuard, run_pch
    m, g = load_golden("icosphere1280_s85")
    with pytest.raises(EngineGuard):
        run_pch(m, g["sources"], EngineConfig(max_iterations=0))
    d, st = run_pch(m, g["sources"], EngineConfig(max_iterations=None))
    assert max_rel_dev(d, g["ich_dist"]) <= TOL
    d, _ = run_pch(m, g["sources"], EngineConfig(max_iterations=st.iterations))
    assert max_rel_dev(d, g["ich_dist"]) <= TOL


def test_phase_times_reported():
    """RunStats.time_select / _propagate / _compact / _events (reference
    engine.py:470-473) with phase_times=True: positive, summing to the
    kernel time; zero (not measured) by default."""
    _gpu()
    from paper_1305_1293_b200 import EngineConfig, run_pch
    m, g = load_golden("icosphere20480_s1370")
    _, st = run_pch(m, g["sources"], EngineConfig(phase_times=True))
    parts = [st.time_select, st.time_propagate, st.time_compact, st.time_events]
    assert all(x >= 0.0 for x in parts) and st.time_propagate > 0.0
    assert abs(sum(parts) * 1e3 - st.time_kernel_ms) <= 1e-6 * max(st.time_kernel_ms, 1.0) + 1e-9
    assert st.prop_item_us > 0.0
    _, st0 = run_pch(m, g["sources"])
    assert st0.time_propagate == 0.0


def test_fields_returned_in_independent_host_buffers():
    """run_pch hands back its field in page-locked host memory from a
    caching allocator (engine.py _host_field): every result must stay its
    own buffer -- a later solve, or dropping an earlier result, never
    rewrites a field the caller still holds (views included)."""
    _gpu()
    from paper_1305_1293_b200 import run_pch
    m, g = load_golden("icosphere5120_multi16")
    a, _ = run_pch(m, [0])
    a_copy = a.copy()
    view = a[10:20]
    for s in (1, 2, 3):
        b, _ = run_pch(m, [s])
        assert not np.shares_memory(a, b)
        del b
    del a
    c, _ = run_pch(m, [4])
    assert np.array_equal(view, a_copy[10:20])
    assert c.dtype == np.float64 and c.shape == (m.n_vertices,) and c.flags.writeable
