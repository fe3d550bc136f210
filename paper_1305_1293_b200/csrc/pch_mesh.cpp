// pch_mesh.cpp -- native half-edge construction (host side of the boundary).
//
// Builds the arrays of the reference's SurfaceMesh (reference
// pkg/src/pargeo/mesh.py:44) from vertex positions and triangles, with the
// reference's validation and error messages (mesh.py:142-227).  The
// arithmetic that feeds the solver is arranged to give bit-identical
// values to the reference's numpy expressions -- edge lengths
// sqrt((dx*dx + dy*dy) + dz*dz), corner angles acos of the law-of-cosines
// ratio, total angles accumulated in half-edge order -- so window-level
// parity with the reference holds (compiled with -ffp-contract=off).  The
// arccos itself is left to the caller when `corner_cos_only` is set: numpy's
// vectorised arccos and the C library's differ in the last bit, and the
// corner angles feed the saddle classification and the fan tables.
//
// Twins are found through one sort of the directed-edge keys (origin, dest);
// the reversed key of every half-edge is then a binary search.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/pch_b200.h"

namespace {

constexpr double EPS_ANGLE = 1e-9;        // mesh.py:19
constexpr double EPS_DEGENERATE = 1e-12;  // mesh.py:20
constexpr double TWO_PI = 6.283185307179586;
thread_local std::string g_mesh_err;

int merr(const char *msg) {
    g_mesh_err = msg;
    return PCH_ERR_MESH;
}

}  // namespace

extern "C" {

const char *pch_half_edge_error(void) { return g_mesh_err.c_str(); }

int pch_half_edge_build(const double *positions, int64_t n_vertices, const int64_t *faces, int64_t n_faces,
                        int64_t *origin, int64_t *opposite, double *length, double *corner_angle,
                        double *total_angle, uint8_t *vertex_class, int64_t *outgoing, uint8_t *on_boundary,
                        int32_t corner_cos_only) {
    if (n_faces <= 0) return merr("mesh has no faces");
    const int64_t nhe = 3 * n_faces;
    for (int64_t i = 0; i < nhe; ++i)
        if (faces[i] < 0 || faces[i] >= n_vertices) return merr("face index out of range");
    for (int64_t f = 0; f < n_faces; ++f) {
        const int64_t a = faces[3 * f], b = faces[3 * f + 1], c = faces[3 * f + 2];
        if (a == b || b == c || c == a) return merr("face repeats a vertex");
    }
    // half-edge 3f+k runs faces[f][k] -> faces[f][(k+1) % 3]
    for (int64_t h = 0; h < nhe; ++h) {
        const int64_t f = h / 3, k = h % 3;
        const int64_t u = faces[h], v = faces[3 * f + (k + 1) % 3];
        origin[h] = u;
        const double dx = positions[3 * v] - positions[3 * u];
        const double dy = positions[3 * v + 1] - positions[3 * u + 1];
        const double dz = positions[3 * v + 2] - positions[3 * u + 2];
        length[h] = std::sqrt((dx * dx + dy * dy) + dz * dz);
        if (!(length[h] > 0.0)) return merr("zero-length edge");
    }
    for (int64_t f = 0; f < n_faces; ++f) {
        double l[3] = {length[3 * f], length[3 * f + 1], length[3 * f + 2]};
        std::sort(l, l + 3);
        if (l[0] + l[1] - l[2] <= EPS_DEGENERATE * l[2])
            return merr("degenerate triangle (triangle inequality violated)");
    }
    // twins: sort directed keys, look up each reversed key
    std::vector<std::pair<int64_t, int64_t>> keys(nhe);
    auto dest = [&](int64_t h) { return faces[3 * (h / 3) + (h % 3 + 1) % 3]; };
    for (int64_t h = 0; h < nhe; ++h) keys[h] = {origin[h] * n_vertices + dest(h), h};
    std::sort(keys.begin(), keys.end());
    for (int64_t i = 1; i < nhe; ++i)
        if (keys[i].first == keys[i - 1].first) return merr("non-manifold edge or inconsistent face orientation");
    for (int64_t h = 0; h < nhe; ++h) {
        const int64_t rk = dest(h) * n_vertices + origin[h];
        auto it = std::lower_bound(keys.begin(), keys.end(), std::make_pair(rk, (int64_t)INT64_MIN));
        opposite[h] = (it != keys.end() && it->first == rk) ? it->second : -1;
    }
    // outgoing: the lowest-index outgoing half-edge, or on a boundary the
    // boundary half-edge (clockwise-most: one counterclockwise walk covers
    // the fan, mesh.py:213)
    for (int64_t v = 0; v < n_vertices; ++v) outgoing[v] = -1;
    for (int64_t h = nhe - 1; h >= 0; --h) outgoing[origin[h]] = h;
    std::memset(on_boundary, 0, n_vertices);
    std::vector<uint8_t> seen(n_vertices, 0);
    for (int64_t h = 0; h < nhe; ++h) {
        if (opposite[h] >= 0) continue;
        const int64_t u = origin[h];
        on_boundary[u] = on_boundary[dest(h)] = 1;
        if (seen[u]) return merr("non-manifold vertex (multiple boundary fans)");
        seen[u] = 1;
        outgoing[u] = h;
    }
    // corner angle at origin[h] inside its face, law of cosines (mesh.py:123)
    for (int64_t f = 0; f < n_faces; ++f) {
        const double *l3 = length + 3 * f;
        for (int k = 0; k < 3; ++k) {
            const double out = l3[k], in = l3[(k + 2) % 3], far = l3[(k + 1) % 3];
            double c = (out * out + in * in - far * far) / (2.0 * out * in);
            c = c < -1.0 ? -1.0 : (c > 1.0 ? 1.0 : c);
            corner_angle[3 * f + k] = corner_cos_only ? c : std::acos(c);
        }
    }
    if (corner_cos_only) return PCH_OK;  // the caller finishes the angles
    std::memset(total_angle, 0, sizeof(double) * n_vertices);
    for (int64_t h = 0; h < nhe; ++h) total_angle[origin[h]] += corner_angle[h];
    for (int64_t v = 0; v < n_vertices; ++v)
        vertex_class[v] = total_angle[v] < TWO_PI - EPS_ANGLE ? 0 : (total_angle[v] > TWO_PI + EPS_ANGLE ? 2 : 1);
    return PCH_OK;
}

}  // extern "C"
