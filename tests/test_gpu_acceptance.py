"""The reference's acceptance criteria (pkg/tests/test_acceptance.py) run
against the B200 engine.  Criteria 1, 3, 7 and 8 live in
test_gpu_parity.py; this file covers 2 (cross-engine equality over the
k / selection-mode grid), 4 (Euclidean <= geodesic <= Dijkstra, edge
Lipschitz), 5 (window overhead at the fastest k) and 6 (window count
grows with k)."""
import numpy as np
import pytest

from conftest import TOL, load_golden, max_rel_dev

pytestmark = pytest.mark.gpu

K_GRID = (256, 4096, 16384)
MODES = ("exact", "approximate_strided")


def _gpu():
    from paper_1305_1293_b200 import _native
    if _native.load().pch_device_count() < 1:
        pytest.fail("no CUDA device visible")


def _dijkstra(mesh, src):
    from scipy.sparse import csr_matrix
    from scipy.sparse.csgraph import dijkstra
    n = mesh.n_vertices
    u = mesh.origin
    v = mesh.origin[3 * (np.arange(len(u)) // 3) + (np.arange(len(u)) + 1) % 3]
    g = csr_matrix((mesh.length, (u, v)), shape=(n, n))
    return dijkstra(g, directed=False, indices=src)


@pytest.mark.parametrize("name", ["icosphere320_s21", "icosphere1280_s85", "icosphere5120_s342",
                                  "icosphere20480_s1370", "bumpy_sphere20k_s3",
                                  "bumpy_torus4800_s5", "disk_patch_s2000"])
def test_criterion_2_cross_engine_grid(name):
    _gpu()
    from paper_1305_1293_b200 import EngineConfig, run_pch
    m, g = load_golden(name)
    worst = 0.0
    for k in K_GRID:
        for mode in MODES:
            for det in (False, True):
                d, _ = run_pch(m, g["sources"], EngineConfig(k=k, selection_mode=mode,
                                                             deterministic=det))
                dev = max_rel_dev(d, g["ich_dist"])
                assert dev <= TOL, (name, k, mode, det, dev)
                worst = max(worst, dev)
    print(f"{name}: worst rel dev {worst:.2e}")


@pytest.mark.parametrize("name", ["tiny_cube_s0", "tiny_octahedron_s0", "tiny_saddle8_s4",
                                  "tiny_torus4x6_s12", "icosphere5120_s342",
                                  "bumpy_sphere20k_s3", "bumpy_torus4800_s5", "disk_patch_s0"])
def test_criterion_4_sandwich_and_lipschitz(name):
    _gpu()
    from paper_1305_1293_b200 import run_pch
    m, g = load_golden(name)
    src = int(g["sources"][0])
    d, _ = run_pch(m, [src])
    chord = np.linalg.norm(m.positions - m.positions[src], axis=1)
    upper = _dijkstra(m, src)
    assert np.all(d >= chord - TOL)
    fin = np.isfinite(upper)
    assert np.all(d[fin] <= upper[fin] + TOL)
    dest = m.origin[3 * (np.arange(m.n_half_edges) // 3) + (np.arange(m.n_half_edges) + 1) % 3]
    assert np.all(np.abs(d[m.origin] - d[dest]) <= m.length + TOL)


def test_criteria_5_6_window_count_vs_k():
    """Window overhead vs the sequential engine at the fastest k of the
    sweep (<= 1.5x, criterion 5) and monotone growth of the window count
    with k (Spearman >= 0.9, criterion 6), on the 20k-face icosphere."""
    _gpu()
    from scipy.stats import spearmanr
    from paper_1305_1293_b200 import EngineConfig, run_pch
    m, g = load_golden("icosphere20480_s1370")
    ich_windows = int(g["ich_windows"])
    ks = [2 ** e for e in range(8, 17)]
    windows, times, det_windows, exact_windows = [], [], [], []
    for k in ks:
        best = None
        for _ in range(3):
            _, st = run_pch(m, g["sources"], EngineConfig(k=k))
            best = st if best is None or st.time_kernel_ms < best.time_kernel_ms else best
        windows.append(best.total_windows_created)
        times.append(best.time_kernel_ms)
        # the k trend on the reproducible (deterministic) schedule
        det_windows.append(run_pch(m, g["sources"],
                                   EngineConfig(k=k, deterministic=True,
                                                selection_mode="approximate_strided"))[1].total_windows_created)
        exact_windows.append(run_pch(m, g["sources"],
                                     EngineConfig(k=k, deterministic=True))[1].total_windows_created)
    rho = float(spearmanr(ks, det_windows).statistic)
    rho_exact = float(spearmanr(ks, exact_windows).statistic)
    fastest = int(np.argmin(times))
    ratio = windows[fastest] / ich_windows
    print(f"k={ks[fastest]} fastest ({times[fastest]:.2f} ms), windows x{ratio:.3f} of ICH; "
          f"Spearman {rho:.3f} (approximate_strided), {rho_exact:.3f} (exact: {exact_windows})")
    assert rho >= 0.9
    # exact selection: the same trend; above k = 8192 the whole pool is
    # selected (counts tie) and the last partial selection can sit within
    # a few hundred windows (0.02 %) of the saturated count, which flips a
    # rank -- so monotonicity is checked to that tolerance
    assert all(b >= a * (1 - 2e-4) for a, b in zip(exact_windows, exact_windows[1:]))
    assert exact_windows[-1] > exact_windows[0]
    assert ratio <= 1.5
