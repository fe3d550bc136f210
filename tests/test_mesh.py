"""Host mesh construction (the data format feeding the device path);
mirrors the reference's mesh tests (reference tests/test_mesh.py)."""
import math

import numpy as np
import pytest

from paper_1305_1293_b200 import meshes
from paper_1305_1293_b200.mesh import (BOUNDARY, MeshError, VertexClass,
                                       build_half_edge_mesh,
                                       classify_total_angle, next_half_edge,
                                       prev_half_edge)


@pytest.mark.parametrize("j,expected", [(4, 5), (5, 3), (0, 1)])
def test_next_half_edge(j, expected):
    assert next_half_edge(j) == expected


def test_prev_inverts_next():
    for j in range(60):
        assert prev_half_edge(next_half_edge(j)) == j


def test_single_triangle():
    m = meshes.make("triangle")
    assert m.n_half_edges == 3
    np.testing.assert_allclose(sorted(m.length), [1.0, 1.0, math.sqrt(2.0)])
    assert np.all(m.opposite == BOUNDARY)


def test_cube_structure(cube):
    assert cube.n_half_edges == 36
    assert np.all(cube.opposite >= 0)
    assert np.all(cube.vertex_class == VertexClass.SPHERICAL)
    np.testing.assert_allclose(cube.total_angle, 1.5 * math.pi)


def test_classification_examples():
    grid = build_half_edge_mesh(*meshes.grid(4, 4))
    center = 2 * 5 + 2
    assert grid.classify_vertex(center) is VertexClass.EUCLIDEAN
    fan8 = build_half_edge_mesh(*meshes.saddle_fan(8))
    assert fan8.classify_vertex(0) is VertexClass.SADDLE
    assert abs(fan8.total_angle[0] - 8 * math.pi / 3) < 1e-9


def test_classify_total_angle_band():
    two_pi = 2 * math.pi
    assert classify_total_angle(two_pi - 1e-6) is VertexClass.SPHERICAL
    assert classify_total_angle(two_pi + 1e-6) is VertexClass.SADDLE
    assert classify_total_angle(two_pi + 1e-12) is VertexClass.EUCLIDEAN


def _face_scan_neighbors(faces, v):
    return {int(u) for tri in faces if v in tri for u in tri if u != v}


def test_one_ring_matches_face_scan(tiny_corpus):
    for name, m in tiny_corpus.items():
        for v in range(m.n_vertices):
            assert set(m.one_ring(v)) == _face_scan_neighbors(m.faces, v), (name, v)


def test_opposite_involution_and_lengths(tiny_corpus):
    for name, m in tiny_corpus.items():
        o = m.opposite
        inner = np.where(o >= 0)[0]
        assert np.array_equal(o[o[inner]], inner), name
        assert np.array_equal(m.length[inner], m.length[o[inner]]), name


def test_corner_angles_sum_to_pi(tiny_corpus):
    for name, m in tiny_corpus.items():
        np.testing.assert_allclose(m.corner_angle.reshape(-1, 3).sum(1), math.pi, atol=1e-9)


def test_boundary_outgoing_is_clockwise_most():
    m = build_half_edge_mesh(*meshes.grid(3, 3))
    for v in np.where(m.on_boundary)[0]:
        h = m.outgoing[v]
        assert m.opposite[h] == BOUNDARY  # the walk starts on the boundary


@pytest.mark.parametrize("faces,msg", [
    ([[0, 1, 1]], "repeats a vertex"),
    ([[0, 1, 5]], "out of range"),
    ([[0, 1, 2], [0, 1, 2]], "non-manifold"),
])
def test_mesh_errors(faces, msg):
    p = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0]], float)
    with pytest.raises(MeshError, match=msg):
        build_half_edge_mesh(p, faces)


def test_degenerate_triangle_rejected():
    p = np.array([[0, 0, 0], [1, 0, 0], [2, 0, 0]], float)
    with pytest.raises(MeshError, match="degenerate"):
        build_half_edge_mesh(p, [[0, 1, 2]])


def test_build_matches_reference_arithmetic_bitwise():
    """The host arrays fed to the device must equal the reference's bit
    for bit (checked against the golden fixture's regenerated mesh)."""
    from conftest import load_golden
    m, g = load_golden("bumpy_sphere20k_s3")
    p, f = g["positions"], g["faces"]
    vec = p[np.roll(f, -1, axis=1).reshape(-1)] - p[f.reshape(-1)]
    assert np.array_equal(m.length, np.sqrt(np.sum(vec * vec, axis=1)))


def test_native_builder_bitwise_matches_reference():
    """The native construction (pch_half_edge_build) reproduces the
    reference's SurfaceMesh arrays bit for bit (fixtures made by the
    reference itself, tests/golden/make_mesh_golden.py)."""
    import os
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "mesh_arrays.npz"))
    names = sorted({k.split("/")[0] for k in g.files})
    assert names
    for name in names:
        m = build_half_edge_mesh(g[f"{name}/positions"], g[f"{name}/faces"])
        for k in ("origin", "opposite", "length", "corner_angle", "total_angle", "vertex_class",
                  "outgoing", "on_boundary"):
            assert np.array_equal(getattr(m, k), g[f"{name}/{k}"]), (name, k)
