import glob
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")
TOL = 1e-9  # north star: max relative per-vertex error vs the CPU oracle


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running (large meshes)")


def max_rel_dev(a, b, floor=1e-12):
    """Largest relative deviation, requiring identical infinity flags
    (reference tests/conftest.py:47)."""
    a = np.asarray(a)
    b = np.asarray(b)
    if not np.array_equal(np.isfinite(a), np.isfinite(b)):
        return np.inf
    both = np.isfinite(a)
    if not both.any():
        return 0.0
    return float(np.max(np.abs(a[both] - b[both]) / np.maximum(np.abs(b[both]), floor)))


@pytest.fixture(scope="session")
def rel_dev():
    return max_rel_dev


def golden_cases():
    """Reference-generated fixtures (make_golden.py); the large_* oracle
    fixtures of the configuration meshes (make_large.py) are separate."""
    return sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "*.npz"))
                  if not os.path.basename(p).startswith(("large_", "mesh_arrays")))


def load_golden(name):
    from paper_1305_1293_b200.mesh import build_half_edge_mesh
    g = dict(np.load(os.path.join(GOLDEN, name + ".npz")))
    return build_half_edge_mesh(g["positions"], g["faces"]), g


@pytest.fixture(scope="session")
def tiny_corpus():
    from paper_1305_1293_b200 import meshes
    return meshes.tiny_corpus()


@pytest.fixture(scope="session")
def cube():
    from paper_1305_1293_b200 import meshes
    return meshes.make("cube")


@pytest.fixture(scope="session")
def icospheres():
    from paper_1305_1293_b200 import meshes
    from paper_1305_1293_b200.mesh import build_half_edge_mesh
    return {20 * 4 ** s: build_half_edge_mesh(*meshes.normalize_edge_scale(*meshes.icosphere(s)))
            for s in (2, 3, 4, 5)}
