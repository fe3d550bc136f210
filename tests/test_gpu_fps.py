"""Farthest-point sampling on the device (include/pch_b200.h: pch_fps;
north star: batched multi-source workloads).  The reference has no FPS
entry point; the composition it replaces is a loop of run_pch calls with a
host argmax, so the checker here is the CPU oracle's run_ich per sample,
min-combined (engine.py:433 semantics: a multi-source field is the
pointwise minimum of the single-source fields).

Greedy picks are checked tie-robustly: at every step the chosen vertex's
oracle min-field distance must equal the oracle maximum to TOL (an exact
tie may legitimately resolve either way between two fp64 evaluations)."""
import numpy as np
import pytest

from conftest import TOL, load_golden, max_rel_dev

pytestmark = pytest.mark.gpu


def _gpu():
    from paper_1305_1293_b200 import _native
    if _native.load().pch_device_count() < 1:
        pytest.fail("no CUDA device visible")


def _check_greedy(m, samples, field):
    from oracle import oracle as O
    dmin = None
    for s, v in enumerate(samples):
        if s > 0:
            best = np.max(dmin)
            assert dmin[v] >= best * (1 - TOL), (s, int(v), float(dmin[v]), float(best))
        f, _ = O.run_ich(m, [int(v)])
        dmin = f if dmin is None else np.minimum(dmin, f)
    assert max_rel_dev(field, dmin) <= TOL
    return dmin


# closed surfaces: greedy picks land on boundaries of open meshes, where
# the reference's own engines disagree on shadowed vertices
@pytest.mark.parametrize("name,n", [("bumpy_sphere20k_s3", 12), ("bumpy_torus4800_s5", 10),
                                    ("icosphere5120_s342", 8), ("icosphere1280_s85", 16),
                                    ("tiny_torus4x6_s0", 6)])
def test_fps_greedy_matches_oracle(name, n):
    _gpu()
    from paper_1305_1293_b200 import farthest_point_sampling
    m, g = load_golden(name)
    first = int(g["sources"][0])
    samples, field, st = farthest_point_sampling(m, n, first)
    assert samples[0] == first
    assert len(samples) == n and st.iterations > 0
    _check_greedy(m, samples, field)


def test_fps_field_is_multi_source_field():
    """The final min-field equals one multi-source run over the samples."""
    _gpu()
    from paper_1305_1293_b200 import farthest_point_sampling, run_pch
    m, g = load_golden("bumpy_sphere20k_s3")
    samples, field, _ = farthest_point_sampling(m, 20, 7)
    multi, _ = run_pch(m, samples)
    assert max_rel_dev(field, multi) <= TOL
    assert len(set(samples.tolist())) == len(samples)  # a closed surface never repeats


def test_fps_single_sample_is_single_field():
    _gpu()
    from paper_1305_1293_b200 import farthest_point_sampling, run_pch
    m, g = load_golden("icosphere5120_s342")
    samples, field, _ = farthest_point_sampling(m, 1, 342)
    single, _ = run_pch(m, [342])
    assert samples.tolist() == [342]
    assert np.array_equal(field, single) or max_rel_dev(field, single) <= TOL


def test_fps_seeded_solves_prune():
    """Seeding with the min-field so far makes later samples cheap: the
    whole 16-sample run propagates far fewer windows than 16 fields."""
    _gpu()
    from paper_1305_1293_b200 import farthest_point_sampling, run_pch
    m, g = load_golden("bumpy_sphere20k_s3")
    _, _, st = farthest_point_sampling(m, 16, 0)
    _, one = run_pch(m, [0])
    assert st.windows_propagated < 6 * one.windows_propagated


def test_fps_deterministic_mode_bitwise():
    _gpu()
    from paper_1305_1293_b200 import EngineConfig, farthest_point_sampling
    m, _ = load_golden("bumpy_torus4800_s5")
    cfg = EngineConfig(deterministic=True)
    a = farthest_point_sampling(m, 8, 3, cfg)
    b = farthest_point_sampling(m, 8, 3, cfg)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    _check_greedy(m, a[0], a[1])


def test_fps_errors():
    _gpu()
    from paper_1305_1293_b200 import farthest_point_sampling
    m, _ = load_golden("tiny_cube_s0")
    with pytest.raises(ValueError):
        farthest_point_sampling(m, 0, 0)
    with pytest.raises(ValueError):
        farthest_point_sampling(m, 3, m.n_vertices)
    with pytest.raises(ValueError):
        farthest_point_sampling(m, 3, -1)
