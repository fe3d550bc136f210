"""GPU parity on the BASELINE.json configuration meshes (configs[1]-[4]).

Fixtures: tests/golden/large_*.npz, made once by tests/golden/make_large.py
from the sequential ICH restatement in oracle/ (reference engine.py:624,
pinned to the reference itself by tests/test_oracle_golden.py).  They hold
the oracle's complete unreachable set and a seeded sample of its distances.

Two oracle fields per case: the reference's default configuration (fan
clip) and its fan_mode="full_edges" (every saddle wedge emitted, then
filtered).  On these meshes the default one has rounding holes and a few
detoured vertices (thin fans of nearly flat saddles dropped by the absolute
tiny-window rule); the full-fan field has neither, and is
the reference answer.  The rule checked:
  * every vertex the full-fan oracle reaches, the GPU reaches;
  * on the sampled vertices: relative error <= 1e-9 against the full-fan
    oracle, and never longer than the default-mode oracle by more than
    1e-9 (the GPU may only be shorter where the reference detoured);
  * size-independent properties of the full GPU field: edge-Lipschitz
    (|d(u) - d(v)| <= |uv|) on every edge with both ends reached, the
    Euclidean lower bound d(v) >= |p(v) - p(s)|, d(s) = 0.
"""
import os

import numpy as np
import pytest

from conftest import GOLDEN, TOL

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

ROWS = [f"torus500k_row{i}" for i in range(10)]

_MESHES = {}


def _mesh(name):
    from paper_1305_1293_b200 import meshes
    if name not in _MESHES:
        _MESHES.clear()  # one large mesh resident at a time (host and device)
        _MESHES[name] = meshes.bench_mesh(name)
    return _MESHES[name]


def _fixture(case):
    path = os.path.join(GOLDEN, f"large_{case}.npz")
    if not os.path.exists(path):
        pytest.fail(f"missing fixture {path} (tests/golden/make_large.py)")
    g = dict(np.load(path))
    m = _mesh(str(g["mesh"]))
    sig = np.array([m.n_vertices, m.n_faces, float(np.sum(m.length))])
    assert np.allclose(sig, g["mesh_sig"], rtol=1e-12, atol=0), "mesh generator changed"
    return m, g


def field_report(m, d, g):
    """Deviation counts of a GPU field against the fixture's oracles."""
    src = int(g["source"])
    fin = np.isfinite(d)
    if "holes_full" not in g:
        pytest.fail("fixture lacks the full-fan oracle (tests/golden/make_large.py)")
    ref_holes = set(g["holes_full"].tolist())
    gpu_holes = set(np.flatnonzero(~fin).tolist())
    idx, val, vfull = g["idx"], g["val"], g["val_full"]
    rf = np.isfinite(vfull)
    rel = (d[idx[rf]] - vfull[rf]) / np.maximum(vfull[rf], 1e-12)
    rel = np.where(np.isfinite(rel), rel, np.inf)
    cf = np.isfinite(val)
    longer_than_clip = (d[idx[cf]] - val[cf]) / np.maximum(val[cf], 1e-12) > TOL
    u = m.origin
    v = m.origin[3 * (np.arange(len(u)) // 3) + (np.arange(len(u)) + 1) % 3]
    both = fin[u] & fin[v]
    gap = np.abs(d[u] - d[v]) - m.length * (1 + 1e-12)
    dmax = float(np.max(d[fin])) if fin.any() else 1.0
    lip_bad = np.unique(np.concatenate([u[both & (gap > 1e-9 * max(1.0, dmax))],
                                        v[both & (gap > 1e-9 * max(1.0, dmax))]]))
    chord = np.linalg.norm(m.positions - m.positions[src], axis=1)
    return {"source_zero": bool(d[src] == 0.0),
            "gpu_only_holes": sorted(gpu_holes - ref_holes),
            "max_rel_err": float(np.max(np.abs(rel))) if rel.size else 0.0,
            "n_off": int(np.sum(np.abs(rel) > TOL)),
            "n_longer_than_clip": int(np.sum(longer_than_clip)),
            "lipschitz_vertices": lip_bad.tolist(),
            "below_euclid": int(np.sum(d[fin] < chord[fin] * (1 - 1e-12) - 1e-9)),
            "holes_gpu": len(gpu_holes), "holes_clip": int(len(g["holes"])),
            "filled_vs_clip": len(set(g["holes"].tolist()) - gpu_holes)}


def check_field(m, d, g, label):
    """The strict rule above."""
    assert d.shape == (m.n_vertices,)
    r = field_report(m, d, g)
    assert r["source_zero"], label
    assert not r["gpu_only_holes"], f"{label}: unreached vertices {r['gpu_only_holes'][:10]}"
    assert r["max_rel_err"] <= TOL, f"{label}: max relative error {r['max_rel_err']:.3e}"
    assert r["n_longer_than_clip"] == 0, label
    assert not r["lipschitz_vertices"], f"{label}: edge-Lipschitz violated at {r['lipschitz_vertices'][:10]}"
    assert r["below_euclid"] == 0, label
    return r


@pytest.mark.parametrize("case", ["terrain1m", "torus500k", "sphere16m"])
@pytest.mark.parametrize("deterministic", [False, True])
def test_config_single_source(case, deterministic):
    from paper_1305_1293_b200 import EngineConfig, run_pch
    if deterministic and case == "sphere16m":
        pytest.skip("two-barrier solver on the 16M mesh: tools/bigcheck.py")
    m, g = _fixture(case)
    d, st = run_pch(m, [int(g["source"])], EngineConfig(deterministic=deterministic))
    rep = check_field(m, d, g, case)
    assert st.iterations > 0 and st.total_windows_created > 0
    print(case, "det" if deterministic else "live", rep, f"{st.time_kernel_ms:.2f} ms")


@pytest.mark.parametrize("case", ["knot1m", "knotg1m"])
@pytest.mark.parametrize("mode", ["default", "deterministic_margin"])
def test_config_knot1m(case, mode):
    """configs[2] at a quarter size (1M-face torus knot, same skinny tube):
    small enough for the oracle's full-fan mode, so the strict rule holds
    against the reference answer.  The reference's default mode leaves
    rounding holes and detoured vertices here too.  knotg1m: the same tube
    with six bridges between its strands (genus 7, configs[2]'s
    "high-genus")."""
    from paper_1305_1293_b200 import EngineConfig, run_pch
    m, g = _fixture(case)
    cfg = EngineConfig() if mode == "default" else EngineConfig(deterministic=True, fan_margin=1e-5)
    d, st = run_pch(m, [int(g["source"])], cfg)
    rep = check_field(m, d, g, f"{case} {mode}")
    print(case, mode, {k: (v if not isinstance(v, list) else len(v)) for k, v in rep.items()},
          f"{st.time_kernel_ms:.1f} ms")


def test_config_knot1m_absolute_tiny_rule_reproduces_the_defect():
    """The round-1 knot defect, reproduced on the 1M-face knot: with the
    reference's absolute tiny-window rule the thin fans of nearly flat
    saddles are dropped and the one-barrier solver leaves vertices
    unreached or reaches them along detours (measured: 215 unreached, 182
    up to 6 % long); the default angular rule reaches all of them exactly
    (test_config_knot1m)."""
    from paper_1305_1293_b200 import EngineConfig, run_pch
    m, g = _fixture("knot1m")
    d, _ = run_pch(m, [int(g["source"])], EngineConfig(tiny_rule="absolute"))
    r = field_report(m, d, g)
    print("knot1m absolute", {k: (v if not isinstance(v, list) else len(v)) for k, v in r.items()})
    assert len(r["gpu_only_holes"]) > 0 or r["n_off"] > 0


def _brief(r):
    """A report with its vertex lists replaced by their lengths (printing)."""
    if isinstance(r, dict):
        return {k: _brief(v) for k, v in r.items()}
    return len(r) if isinstance(r, list) else r


def _knot4m_report(m, d, g):
    """The 4M-face knots against the default-mode oracle, one-sidedly --
    never longer on a sampled vertex, shorter only where the oracle
    detoured -- plus the full-field properties; the full-fan oracle's
    deviations (field_report) ride along where the fixture holds it."""
    src = int(g["source"])
    fin = np.isfinite(d)
    idx, val = g["idx"], g["val"]
    cf = np.isfinite(val)
    rel = (d[idx[cf]] - val[cf]) / np.maximum(val[cf], 1e-12)
    u = m.origin
    v = m.origin[3 * (np.arange(len(u)) // 3) + (np.arange(len(u)) + 1) % 3]
    both = fin[u] & fin[v]
    gap = np.abs(d[u] - d[v]) - m.length * (1 + 1e-12)
    lip = np.unique(np.concatenate([u[both & (gap > 1e-9 * float(np.max(d[fin])))],
                                    v[both & (gap > 1e-9 * float(np.max(d[fin])))]]))
    chord = np.linalg.norm(m.positions - m.positions[src], axis=1)
    return {"source_zero": bool(d[src] == 0.0), "holes_gpu": int((~fin).sum()),
            "holes_oracle": int(len(g["holes"])),
            "unreached_oracle_reached": int(np.sum(~np.isfinite(d[idx[cf]]))),
            "n_longer": int(np.sum(rel > TOL)), "n_shorter": int(np.sum(rel < -TOL)),
            "n_sample": int(cf.sum()), "max_longer": float(max(rel.max(), 0.0)),
            "lipschitz_vertices": lip.tolist(),
            "below_euclid": int(np.sum(d[fin] < chord[fin] * (1 - 1e-12) - 1e-9)),
            "full": field_report(m, d, g) if "holes_full" in g else None}


@pytest.mark.parametrize("case", ["knot4m", "knotg4m"])
def test_config_knot4m_exact(case):
    """configs[2], the 4M-face torus knot, in the configuration exact on it
    (two-barrier solver, 1e-4 rad fan margin; 27 s): the
    strict rule against the reference's full-fan oracle where the fixture
    holds it (2.4 h of oracle CPU time each; measured max relative error
    1.2e-14 / 1.3e-14, every vertex reached); otherwise every vertex reached, never
    longer than the reference's default mode on any sampled vertex, shorter
    only on the few it detoured, edge-Lipschitz everywhere."""
    from paper_1305_1293_b200 import EngineConfig, run_pch
    m, g = _fixture(case)
    d, st = run_pch(m, [int(g["source"])], EngineConfig(deterministic=True, fan_margin=1e-4))
    r = _knot4m_report(m, d, g)
    print(case, "exact", _brief(r),
          f"{st.time_kernel_ms:.1f} ms")
    if r["full"] is not None:  # the strict rule against the reference answer
        check_field(m, d, g, f"{case} exact")
    assert r["source_zero"] and r["below_euclid"] == 0
    assert r["holes_gpu"] == 0
    assert r["n_longer"] == 0
    assert r["n_shorter"] <= 0.002 * r["n_sample"]
    assert not r["lipschitz_vertices"]


@pytest.mark.parametrize("case", ["knot4m", "knotg4m"])
@pytest.mark.parametrize("fan_mode", ["clip", "full_edges"])
def test_config_knot4m_live_residual(case, fan_mode):
    """configs[2] with the fast one-barrier solver: the residual it leaves
    on this ill-conditioned mesh, bounded (measured over
    repeated runs, the solver is not bitwise reproducible).  Default (fan
    clip): 14-17 of 2M vertices unreached, 68-117 vertices in edges that
    break the Lipschitz bound, where the reference's own default mode leaves
    7824 unreached and >= 530 detoured.  full_edges: none unreached, 0-2
    detoured vertices."""
    from paper_1305_1293_b200 import EngineConfig, run_pch
    m, g = _fixture(case)
    d, st = run_pch(m, [int(g["source"])], EngineConfig(fan_mode=fan_mode))
    r = _knot4m_report(m, d, g)
    print(case, "live", fan_mode, _brief(r),
          f"{st.time_kernel_ms:.1f} ms")
    assert r["source_zero"] and r["below_euclid"] == 0
    if fan_mode == "clip":
        assert r["holes_gpu"] <= 64 and r["holes_gpu"] < r["holes_oracle"] // 10
        assert len(r["lipschitz_vertices"]) <= 256
        assert r["n_longer"] <= 3
    else:
        assert r["holes_gpu"] == 0
        assert len(r["lipschitz_vertices"]) <= 8
        assert r["n_longer"] <= 1
    if r["full"] is not None:  # against the full-fan oracle (the reference answer)
        f = r["full"]
        assert len(f["gpu_only_holes"]) == r["holes_gpu"]
        assert f["n_off"] <= (8 if fan_mode == "clip" else 1)
        assert f["n_longer_than_clip"] <= 3


def test_config_rows_torus500k():
    """configs[4]: batched distance-matrix rows on the 500k-face torus; every
    row obeys the rule against its own oracle field, and equals the
    single-source field of the same source on every vertex both reach."""
    from paper_1305_1293_b200 import run_pch, run_pch_rows
    fx = [_fixture(c) for c in ROWS]
    m = fx[0][0]
    src = [int(g["source"]) for _, g in fx]
    rows, st = run_pch_rows(m, src)
    assert rows.shape == (len(src), m.n_vertices)
    for r, (_, g) in enumerate(fx):
        check_field(m, rows[r], g, ROWS[r])
    for r in (1, 2, 4):  # rows where the default-mode oracle has rounding holes
        single, _ = run_pch(m, [src[r]])
        assert np.array_equal(np.isfinite(single), np.isfinite(rows[r]))
        both = np.isfinite(single)
        assert np.max(np.abs(single[both] - rows[r][both]) / np.maximum(single[both], 1e-12)) <= TOL


def test_sphere16m_rows_grow_without_rerun():
    """configs[3] mesh, batched rows from a deliberately small pool: the
    pool grows at iteration boundaries (windows migrated, solve resumed),
    never rerun, and the rows match single-source fields."""
    from paper_1305_1293_b200 import EngineConfig, run_pch, run_pch_rows
    m, g = _fixture("sphere16m")
    src = [int(g["source"]), 17, 4_000_000]
    rows, st = run_pch_rows(m, src, EngineConfig(pool_capacity=1 << 19))
    assert st.buffer_regrows >= 1 and st.pool_restarts == 0
    check_field(m, rows[0], g, "sphere16m row 0")
    one, _ = run_pch(m, [src[2]])
    assert np.array_equal(np.isfinite(one), np.isfinite(rows[2]))
    fin = np.isfinite(one)
    assert np.max(np.abs(rows[2][fin] - one[fin]) / np.maximum(one[fin], 1e-12)) <= TOL
