"""Pin the CPU oracle (oracle/pch_oracle.c) against the reference's own
outputs (tests/golden, produced by tests/golden/make_golden.py from the
reference package).  CPU only."""
import math

import numpy as np
import pytest

from conftest import TOL, golden_cases, load_golden, max_rel_dev
from oracle import oracle as O

CASES = golden_cases()


def test_golden_fixtures_present():
    assert len(CASES) >= 30
    assert sum(c.startswith("tiny_") for c in CASES) >= 20


@pytest.mark.parametrize("name", CASES)
def test_oracle_ich_matches_reference(name):
    m, g = load_golden(name)
    d, st = O.run_ich(m, g["sources"])
    assert max_rel_dev(d, g["ich_dist"]) <= 1e-12, name
    # the restatement follows the reference window by window
    assert st["total_windows_created"] == int(g["ich_windows"]), name
    assert st["windows_propagated"] == int(g["ich_propagated"]), name


@pytest.mark.parametrize("name", [c for c in CASES if c.startswith("tiny_")])
def test_oracle_matches_brute_force(name):
    m, g = load_golden(name)
    d, _ = O.run_ich(m, g["sources"])
    assert max_rel_dev(d, g["brute_dist"]) < TOL, name


@pytest.mark.parametrize("name", CASES)
def test_oracle_pch_matches_reference(name):
    m, g = load_golden(name)
    d, st = O.run_pch(m, g["sources"], k=4096, workers=4)
    assert max_rel_dev(d, g["pch_dist"]) < TOL, name
    if np.array_equal(np.isfinite(g["pch_dist"]), np.isfinite(g["ich_dist"])):
        assert max_rel_dev(d, g["ich_dist"]) < TOL, name


def test_reference_engines_disagree_on_boundary_shadows():
    """Documented reference behaviour: with a non-convex (angle > pi)
    boundary vertex the reference never bends geodesics around it, and
    which shadowed vertices stay unreachable depends on the schedule --
    its own run_pch and run_ich disagree (37 vs 43 unreachable on this
    mesh, and up to ~2.4e-4 relative on vertices both reach).  Parity is
    therefore only defined on meshes without boundary shadows: closed
    meshes and convex planar rims."""
    _, g = load_golden("terrain3200_corner")
    n_pch = int(np.sum(~np.isfinite(g["pch_dist"])))
    n_ich = int(np.sum(~np.isfinite(g["ich_dist"])))
    assert (n_pch, n_ich) == (37, 43)
    both = np.isfinite(g["pch_dist"]) & np.isfinite(g["ich_dist"])
    dev = max_rel_dev(g["pch_dist"][both], g["ich_dist"][both])
    assert 1e-6 < dev < 1e-3


def test_oracle_pch_order_independence():
    m, g = load_golden("icosphere1280_s85")
    base, _ = O.run_pch(m, g["sources"], k=1, workers=1)
    for k, t, mode in ((256, 4, "exact"), (16384, 8, "exact"), (256, 4, "approximate_strided")):
        d, _ = O.run_pch(m, g["sources"], k=k, workers=t, selection_mode=mode)
        assert max_rel_dev(d, base) < TOL


def test_oracle_cube_diagonal():
    m, g = load_golden("tiny_cube_s0")
    d, _ = O.run_ich(m, [0])
    assert d[6] == pytest.approx(math.sqrt(5.0), rel=1e-12)


def test_oracle_unreachable_flags():
    m, g = load_golden("terrain3200_corner")
    d, _ = O.run_ich(m, g["sources"])
    assert np.sum(~np.isfinite(d)) == np.sum(~np.isfinite(g["ich_dist"])) > 0


def test_oracle_iteration_guard():
    m, g = load_golden("icosphere320_s21")
    with pytest.raises(RuntimeError, match="iteration cap"):
        O.run_pch(m, g["sources"], k=1, max_iterations=3)


def test_oracle_rejects_bad_sources():
    m, _ = load_golden("tiny_cube_s0")
    with pytest.raises(ValueError):
        O.run_ich(m, [])
    with pytest.raises(ValueError):
        O.run_pch(m, [99])
