"""Synthetic mesh generators: the reference corpus and the BASELINE.json
benchmark families (small instances)."""
import numpy as np
import pytest

from paper_1305_1293_b200 import meshes
from paper_1305_1293_b200.mesh import VertexClass, build_half_edge_mesh


def test_tiny_corpus_sizes(tiny_corpus):
    assert len(tiny_corpus) >= 10
    assert all(m.n_faces <= 50 for m in tiny_corpus.values())


@pytest.mark.parametrize("sub", [0, 1, 2, 3])
def test_icosphere_counts(sub):
    p, f = meshes.icosphere(sub)
    assert len(f) == 20 * 4 ** sub
    assert len(p) == 10 * 4 ** sub + 2
    np.testing.assert_allclose(np.linalg.norm(p, axis=1), 1.0, atol=1e-12)
    m = build_half_edge_mesh(p, f)
    assert np.all(m.opposite >= 0)


def test_icosphere_matches_reference_golden():
    from conftest import load_golden
    _, g = load_golden("icosphere5120_s342")
    p, f = meshes.normalize_edge_scale(*meshes.icosphere(4))
    assert np.array_equal(f, g["faces"])
    np.testing.assert_allclose(p, g["positions"], rtol=0, atol=1e-12)


def test_terrain_flat_convex_rim():
    p, f = meshes.terrain(40)
    m = build_half_edge_mesh(p, f)
    assert m.n_faces == 2 * 40 * 40
    # every boundary vertex lies on the planar rim with angle <= pi
    b = m.on_boundary
    assert np.all(m.total_angle[b] <= np.pi + 1e-9)
    assert np.ptp(p[b, 2]) == 0.0
    assert np.sum(m.vertex_class == VertexClass.SADDLE) > 0.2 * m.n_vertices
    edge = np.mean(m.length)
    assert abs(edge - 1.0) < 1e-9


def test_torus_knot_tube_closed_and_anisotropic():
    p, f = meshes.torus_knot_tube(n_along=2000, n_around=20)
    m = build_half_edge_mesh(p, f)
    assert m.n_faces == 2 * 2000 * 20
    assert np.all(m.opposite >= 0)  # closed tube
    l3 = m.length.reshape(-1, 3)
    assert np.median(l3.max(1) / l3.min(1)) > 2.0


def test_perturbed_sphere_closed():
    p, f = meshes.perturbed_sphere(12)
    m = build_half_edge_mesh(p, f)
    assert m.n_faces == 6 * 2 * 12 * 12
    assert np.all(m.opposite >= 0)
    # Euler characteristic of a sphere
    n_e = m.n_half_edges // 2
    assert m.n_vertices - n_e + m.n_faces == 2


def test_bench_mesh_names():
    m = meshes.bench_mesh("icosphere20k")
    assert m.n_faces == 20480
    with pytest.raises(KeyError):
        meshes.bench_mesh("nope")
