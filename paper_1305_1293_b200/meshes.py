"""Deterministic synthetic meshes.

The fixed solids and the small corpus mirror the reference generators
(reference ``pkg/src/pargeo/meshes.py``: single_triangle, square, strip,
grid, cube, tetrahedron, octahedron, pyramid, saddle_fan, icosahedron,
icosphere, bumpy_sphere, torus, bumpy_torus, normalize_edge_scale,
tiny_corpus).  The large benchmark meshes named by BASELINE.json's configs
are new here and vectorised so that multi-million-face meshes build in
seconds:

* ``terrain``        — noisy heightfield grid (config 1, ~1M faces)
* ``torus_knot_tube``— tube swept along a (p, q) torus knot with skinny,
                       anisotropic triangles (~4M faces, genus 1)
* ``torus_knot_tube_handles`` — the same tube with bridges between its
                       strands: genus 7 (config 2 as stated, "high-genus")
* ``perturbed_sphere``— subdivided cube-sphere with radial noise
                       (config 3, ~16M faces)

Generators return ``(positions, faces)``; ``make(name)`` builds the
half-edge mesh.
"""
from __future__ import annotations

import math

import numpy as np

from .mesh import SurfaceMesh, build_half_edge_mesh


def single_triangle():
    return (np.array([[0.0, 0.0, 0.0], [1.0, 0.0, 0.0], [0.0, 1.0, 0.0]]),
            np.array([[0, 1, 2]], dtype=np.int64))


def square():
    """Unit square split along its (0,0)-(1,1) diagonal."""
    p = np.array([[0, 0, 0], [1, 0, 0], [1, 1, 0], [0, 1, 0]], dtype=float)
    return p, np.array([[0, 1, 2], [0, 2, 3]], dtype=np.int64)


def strip(n: int, width: float = 1.0):
    """Planar strip of ``n`` unit quads, two triangles each."""
    i = np.arange(n + 1, dtype=float)
    p = np.zeros((2 * (n + 1), 3))
    p[0::2, 0] = i
    p[1::2, 0] = i
    p[1::2, 1] = width
    q = np.arange(n, dtype=np.int64)
    a, b, c, d = 2 * q, 2 * q + 1, 2 * q + 2, 2 * q + 3
    f = np.empty((2 * n, 3), dtype=np.int64)
    f[0::2] = np.stack([a, c, d], 1)
    f[1::2] = np.stack([a, d, b], 1)
    return p, f


def grid(nx: int, ny: int, spacing: float = 1.0, heights=None):
    """Rectangular grid of ``2*nx*ny`` triangles, optionally displaced by
    ``heights(x, y)``; vertex ``(i, j)`` has index ``i*(ny+1)+j``."""
    gx, gy = np.meshgrid(np.arange(nx + 1) * spacing,
                         np.arange(ny + 1) * spacing, indexing="ij")
    gz = np.zeros_like(gx) if heights is None else heights(gx, gy)
    p = np.column_stack([gx.ravel(), gy.ravel(), gz.ravel()])
    i, j = np.meshgrid(np.arange(nx), np.arange(ny), indexing="ij")
    a = (i * (ny + 1) + j).ravel()
    b = ((i + 1) * (ny + 1) + j).ravel()
    f = np.empty((2 * nx * ny, 3), dtype=np.int64)
    f[0::2] = np.stack([a, b, b + 1], 1)
    f[1::2] = np.stack([a, b + 1, a + 1], 1)
    return p, f


def cube():
    p = np.array([[0, 0, 0], [1, 0, 0], [1, 1, 0], [0, 1, 0],
                  [0, 0, 1], [1, 0, 1], [1, 1, 1], [0, 1, 1]], dtype=float)
    f = np.array([[0, 2, 1], [0, 3, 2], [4, 5, 6], [4, 6, 7],
                  [0, 1, 5], [0, 5, 4], [1, 2, 6], [1, 6, 5],
                  [2, 3, 7], [2, 7, 6], [3, 0, 4], [3, 4, 7]], dtype=np.int64)
    return p, f


def tetrahedron():
    p = np.array([[1, 1, 1], [1, -1, -1], [-1, 1, -1], [-1, -1, 1]], float)
    f = np.array([[0, 2, 1], [0, 1, 3], [0, 3, 2], [1, 2, 3]], np.int64)
    return p, f


def octahedron():
    p = np.array([[1, 0, 0], [-1, 0, 0], [0, 1, 0], [0, -1, 0],
                  [0, 0, 1], [0, 0, -1]], dtype=float)
    f = np.array([[0, 2, 4], [2, 1, 4], [1, 3, 4], [3, 0, 4],
                  [2, 0, 5], [1, 2, 5], [3, 1, 5], [0, 3, 5]], np.int64)
    return p, f


def pyramid():
    """Square pyramid closed by a split base."""
    p = np.array([[0, 0, 0], [1, 0, 0], [1, 1, 0], [0, 1, 0],
                  [0.5, 0.5, 0.8]], dtype=float)
    f = np.array([[0, 1, 4], [1, 2, 4], [2, 3, 4], [3, 0, 4],
                  [0, 2, 1], [0, 3, 2]], dtype=np.int64)
    return p, f


def saddle_fan(n: int = 8):
    """``n`` unit equilateral triangles around vertex 0 with the ring
    alternating above/below the plane; a saddle for ``n > 6``."""
    if n < 6 or n % 2:
        raise ValueError("need an even n >= 6 for an equilateral fan")
    rho2 = 0.75 / math.cos(math.pi / n) ** 2
    rho, h = math.sqrt(rho2), math.sqrt(max(1.0 - rho2, 0.0))
    ang = 2.0 * math.pi * np.arange(n) / n
    ring = np.column_stack([rho * np.cos(ang), rho * np.sin(ang),
                            np.where(np.arange(n) % 2 == 0, h, -h)])
    p = np.vstack([[0.0, 0.0, 0.0], ring])
    k = np.arange(n)
    f = np.stack([np.zeros(n, np.int64), 1 + k, 1 + (k + 1) % n], 1)
    return p, f.astype(np.int64)


def icosahedron():
    t = (1.0 + math.sqrt(5.0)) / 2.0
    p = np.array([[-1, t, 0], [1, t, 0], [-1, -t, 0], [1, -t, 0],
                  [0, -1, t], [0, 1, t], [0, -1, -t], [0, 1, -t],
                  [t, 0, -1], [t, 0, 1], [-t, 0, -1], [-t, 0, 1]], float)
    p /= np.linalg.norm(p[0])
    f = np.array([[0, 11, 5], [0, 5, 1], [0, 1, 7], [0, 7, 10], [0, 10, 11],
                  [1, 5, 9], [5, 11, 4], [11, 10, 2], [10, 7, 6], [7, 1, 8],
                  [3, 9, 4], [3, 4, 2], [3, 2, 6], [3, 6, 8], [3, 8, 9],
                  [4, 9, 5], [2, 4, 11], [6, 2, 10], [8, 6, 7], [9, 8, 1]],
                 dtype=np.int64)
    return p, f


def _midpoint_subdivide(p, f, project):
    """One 1-to-4 split; new vertices are numbered in order of first
    appearance of their edge in face order (edges ab, bc, ca)."""
    nv = len(p)
    e = np.stack([f[:, [0, 1]], f[:, [1, 2]], f[:, [2, 0]]], 1).reshape(-1, 2)
    lo, hi = e.min(1), e.max(1)
    key = lo * nv + hi
    uniq, first, inv = np.unique(key, return_index=True, return_inverse=True)
    rank = np.empty(len(uniq), np.int64)
    rank[np.argsort(first, kind="stable")] = np.arange(len(uniq))
    mid_id = nv + rank[inv].reshape(-1, 3)
    ulo, uhi = uniq // nv, uniq % nv
    newp = np.empty((len(uniq), 3))
    newp[rank] = project(p[ulo] + p[uhi])
    ab, bc, ca = mid_id[:, 0], mid_id[:, 1], mid_id[:, 2]
    a, b, c = f[:, 0], f[:, 1], f[:, 2]
    nf = np.stack([np.stack([a, ab, ca], 1), np.stack([b, bc, ab], 1),
                   np.stack([c, ca, bc], 1), np.stack([ab, bc, ca], 1)], 1)
    return np.vstack([p, newp]), nf.reshape(-1, 3)


def icosphere(subdivisions: int):
    """Icosahedron split ``subdivisions`` times onto the unit sphere:
    ``20 * 4**subdivisions`` faces."""
    p, f = icosahedron()
    unit = lambda q: q / np.linalg.norm(q, axis=1, keepdims=True)
    for _ in range(subdivisions):
        p, f = _midpoint_subdivide(p, f, unit)
    return p, f


def bumpy_sphere(subdivisions: int, amplitude: float = 0.12):
    """Icosphere with multi-frequency radial displacement (saddle-rich)."""
    p, f = icosphere(subdivisions)
    x, y, z = p[:, 0], p[:, 1], p[:, 2]
    r = 1.0 + amplitude * (np.sin(5.0 * x + 1.0) * np.sin(4.0 * y + 2.0)
                           + 0.6 * np.sin(7.0 * z + 3.0) * np.sin(3.0 * x)
                           + 0.4 * np.sin(6.0 * y * z + 0.5))
    return p * r[:, None], f


def _wrapped_grid_faces(nu: int, nv: int):
    i, j = np.meshgrid(np.arange(nu), np.arange(nv), indexing="ij")
    a = (i * nv + j).ravel()
    b = (((i + 1) % nu) * nv + j).ravel()
    a2 = (i * nv + (j + 1) % nv).ravel()
    b2 = (((i + 1) % nu) * nv + (j + 1) % nv).ravel()
    f = np.empty((2 * nu * nv, 3), dtype=np.int64)
    f[0::2] = np.stack([a, b, b2], 1)
    f[1::2] = np.stack([a, b2, a2], 1)
    return f


def torus(nu: int, nv: int, major: float = 2.0, minor: float = 0.8):
    """Closed torus with ``2*nu*nv`` faces."""
    a = 2.0 * np.pi * np.arange(nu) / nu
    b = 2.0 * np.pi * np.arange(nv) / nv
    A, B = np.meshgrid(a, b, indexing="ij")
    ring = major + minor * np.cos(B)
    p = np.column_stack([(ring * np.cos(A)).ravel(),
                         (ring * np.sin(A)).ravel(),
                         (minor * np.sin(B)).ravel()])
    return p, _wrapped_grid_faces(nu, nv)


def bumpy_torus(nu: int, nv: int, amplitude: float = 0.25):
    """Torus with radial displacement about its core circle."""
    p, f = torus(nu, nv)
    x, y, z = p[:, 0], p[:, 1], p[:, 2]
    s = 1.0 + amplitude * (np.sin(3.1 * x + 0.7) * np.cos(2.3 * y)
                           + 0.5 * np.sin(4.7 * z + 1.9) * np.sin(1.7 * x))
    ang = np.arctan2(y, x)
    center = np.column_stack([2.0 * np.cos(ang), 2.0 * np.sin(ang),
                              np.zeros_like(x)])
    return center + (p - center) * s[:, None], f


def normalize_edge_scale(positions, faces, target: float = 1.0):
    """Rescale so the mean edge length is ``target`` (the window tolerance
    is absolute, so meshes should have edges of order one)."""
    positions = np.asarray(positions, float)
    faces = np.asarray(faces, np.int64)
    a = positions[faces.ravel()]
    b = positions[faces[:, [1, 2, 0]].ravel()]
    mean_edge = float(np.mean(np.linalg.norm(a - b, axis=1)))
    return positions * (target / mean_edge), faces


# --------------------------------------------------------------------------
# benchmark meshes (BASELINE.json configs)


def terrain(n: int = 708, amplitude: float = 0.35, seed: int = 1305,
            rim: int = 2, ramp: int = 8):
    """Noisy heightfield on an ``n x n`` cell grid (``2 n^2`` faces; n=708
    gives 1,002,528 faces).  Height = smooth multi-octave ridges plus
    per-vertex uniform jitter, in units of the grid spacing, so the
    surface is rough at the triangle scale (plenty of saddles) while every
    triangle stays well shaped.  Heights fade to exactly zero over ``ramp``
    cells and vanish on a ``rim``-cell flat border, so the boundary is a
    planar convex square: no boundary vertex has an interior angle above
    pi, geodesics never need to bend around the boundary, and every
    vertex is reachable (the reference engines only agree on unreachable
    flags for such boundaries).  Mean edge length is
    normalised to one."""
    rng = np.random.default_rng(seed)
    s = 1.0 / max(n, 1)

    def taper(t):
        d = np.minimum(t, n - t)  # cells to the nearest side
        return np.clip((d - rim) / float(max(ramp, 1)), 0.0, 1.0)

    def h(x, y):
        u, v = x * s, y * s
        z = (np.sin(2 * np.pi * (1.3 * u + 0.2)) * np.cos(2 * np.pi * (1.7 * v))
             + 0.5 * np.sin(2 * np.pi * (4.1 * u + 2.9 * v + 0.3))
             + 0.25 * np.sin(2 * np.pi * (9.7 * u - 7.3 * v + 0.7)))
        z = n * 0.02 * z + amplitude * rng.uniform(-1.0, 1.0, x.shape)
        return z * taper(x) * taper(y)

    return normalize_edge_scale(*grid(n, n, 1.0, h))


def torus_knot_tube(p_wind: int = 2, q_wind: int = 3, n_along: int = 20000,
                    n_around: int = 100, tube: float = 0.12):
    """Tube of ``2*n_along*n_around`` faces swept along the (p, q) torus
    knot.  Rings are far denser along the knot than around it, so the
    triangles are skinny and anisotropic (aspect ~ 5-10 at the defaults,
    4M faces), which stresses window-count control."""
    t = 2.0 * np.pi * np.arange(n_along) / n_along

    def curve(tt):
        r = 2.0 + np.cos(q_wind * tt)
        return np.column_stack([r * np.cos(p_wind * tt), r * np.sin(p_wind * tt),
                                -np.sin(q_wind * tt)])

    c = curve(t)
    dt = 1e-4
    tan = curve(t + dt) - curve(t - dt)
    tan /= np.linalg.norm(tan, axis=1, keepdims=True)
    # rotation-minimising-ish frame from a fixed helper axis
    helper = np.array([0.0, 0.0, 1.0])
    nrm = np.cross(tan, helper)
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    bin_ = np.cross(tan, nrm)
    a = 2.0 * np.pi * np.arange(n_around) / n_around
    ca, sa = np.cos(a), np.sin(a)
    wob = 1.0 + 0.15 * np.sin(7.0 * t)[:, None] * np.cos(3.0 * a)[None, :]
    pts = (c[:, None, :] + tube * wob[..., None]
           * (ca[None, :, None] * nrm[:, None, :] + sa[None, :, None] * bin_[:, None, :]))
    return normalize_edge_scale(pts.reshape(-1, 3), _wrapped_grid_faces(n_along, n_around))


def torus_knot_tube_handles(p_wind: int = 2, q_wind: int = 3, n_along: int = 20000,
                            n_around: int = 100, tube: float = 0.12, handles: int = 6,
                            hole_around: int = 6, bridge_rings: int = 24):
    """``torus_knot_tube`` with ``handles`` bridges between strands where
    the knot passes close to itself: genus 1 + handles.  At each site a
    block of tube faces facing the other strand is removed on both strands
    and the two boundary loops are joined by a straight cylinder of
    ``bridge_rings`` rings (only edge lengths matter to the solver, so the
    embedding need not be free of intersections).  The tube keeps its
    skinny, anisotropic triangles; the bridges add long thin ones."""
    t = 2.0 * np.pi * np.arange(n_along) / n_along

    def curve(tt):
        r = 2.0 + np.cos(q_wind * tt)
        return np.column_stack([r * np.cos(p_wind * tt), r * np.sin(p_wind * tt),
                                -np.sin(q_wind * tt)])

    c = curve(t)
    tan = curve(t + 1e-4) - curve(t - 1e-4)
    tan /= np.linalg.norm(tan, axis=1, keepdims=True)
    nrm = np.cross(tan, np.array([0.0, 0.0, 1.0]))
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    bin_ = np.cross(tan, nrm)
    a = 2.0 * np.pi * np.arange(n_around) / n_around
    wob = 1.0 + 0.15 * np.sin(7.0 * t)[:, None] * np.cos(3.0 * a)[None, :]
    pts = (c[:, None, :] + tube * wob[..., None]
           * (np.cos(a)[None, :, None] * nrm[:, None, :] + np.sin(a)[None, :, None] * bin_[:, None, :]))
    # closest approaches of the knot to itself (at least a tenth of the
    # curve apart): local minima of the nearest-strand distance
    m = 2048
    ci = (np.arange(m) * n_along) // m
    cs = c[ci]
    dist = np.linalg.norm(cs[:, None, :] - cs[None, :, :], axis=2)
    sep = np.abs(np.arange(m)[:, None] - np.arange(m)[None, :])
    sep = np.minimum(sep, m - sep)
    dist[sep < m // 10] = np.inf
    nearest = dist.min(axis=1)
    partner = dist.argmin(axis=1)
    minima = [k for k in range(m) if nearest[k] <= nearest[k - 1] and nearest[k] <= nearest[(k + 1) % m]]
    sites, used = [], np.zeros(m, dtype=bool)
    for k in sorted(minima, key=lambda k: nearest[k]):
        if len(sites) == handles:
            break
        kb = int(partner[k])
        if used[k] or used[kb]:
            continue
        for q in (k, kb):
            used[np.arange(q - m // 40, q + m // 40) % m] = True
        sites.append((int(ci[k]), int(ci[kb])))
    # hole size: about square on the tube (along cells are shorter)
    cell_along = np.linalg.norm(c[1] - c[0])
    cell_around = 2.0 * np.pi * tube / n_around
    hole_along = max(2, int(round(hole_around * cell_around / cell_along)))
    removed = np.zeros((n_along, n_around), dtype=bool)  # quad (i, j) removed
    loops = []

    def facing(i, target):
        d = target - c[i]
        ang = np.arctan2(d @ bin_[i], d @ nrm[i])
        return int(round(ang / (2.0 * np.pi) * n_around)) % n_around

    for ia, ib in sites:
        pair = []
        for i_c, other in ((ia, ib), (ib, ia)):
            j_c = facing(i_c, c[other])
            i0, j0 = i_c - hole_along // 2, j_c - hole_around // 2
            for di in range(hole_along):
                for dj in range(hole_around):
                    removed[(i0 + di) % n_along, (j0 + dj) % n_around] = True
            # boundary loop of the hole, counterclockwise in (i, j)
            loop = ([((i0 + k) % n_along, j0 % n_around) for k in range(hole_along)]
                    + [((i0 + hole_along) % n_along, (j0 + k) % n_around) for k in range(hole_around)]
                    + [((i0 + hole_along - k) % n_along, (j0 + hole_around) % n_around)
                       for k in range(hole_along)]
                    + [(i0 % n_along, (j0 + hole_around - k) % n_around) for k in range(hole_around)])
            pair.append([i * n_around + j for i, j in loop])
        loops.append(pair)
    faces = _wrapped_grid_faces(n_along, n_around)
    keep = ~np.repeat(removed.ravel(), 2)
    faces = [faces[keep]]
    positions = [pts.reshape(-1, 3)]
    nv = n_along * n_around
    for la, lb in loops:
        la = np.asarray(la)
        # loop B runs the other way round (the bridge enters the other tube
        # from outside); start it at the vertex nearest loop A's first
        lb = np.asarray(lb)[::-1]
        pa, pb = positions[0][la], positions[0][lb]
        sh = int(np.argmin(np.linalg.norm(pb - pa[0], axis=1)))
        lb, pb = np.roll(lb, -sh), np.roll(pb, -sh, axis=0)
        n = len(la)
        rings = [la]
        for k in range(1, bridge_rings):
            f = k / bridge_rings
            positions.append(pa + f * (pb - pa))
            rings.append(np.arange(nv, nv + n))
            nv += n
        rings.append(lb)
        for r0, r1 in zip(rings[:-1], rings[1:]):
            nx = np.roll(np.arange(n), -1)
            # orientation opposite to the holes' boundary half-edges
            faces.append(np.stack([r0, r0[nx], r1[nx]], 1))
            faces.append(np.stack([r0, r1[nx], r1], 1))
    faces = np.vstack(faces)
    # drop the vertices inside the holes (no face left)
    used = np.zeros(nv, dtype=bool)
    used[faces.ravel()] = True
    remap = np.cumsum(used) - 1
    return normalize_edge_scale(np.vstack(positions)[used], remap[faces])


def perturbed_sphere(n: int = 1155, amplitude: float = 0.04, seed: int = 1293):
    """Cube-sphere: each cube face split into ``n x n`` quads (two
    triangles each; n=1155 gives 16,008,300 faces), projected to the unit
    sphere and displaced radially by smooth bumps plus small jitter."""
    rng = np.random.default_rng(seed)
    # shared vertex lattice on the cube surface: index the (n+1)^3 lattice
    # points that lie on the surface
    g = np.arange(n + 1)
    side = n + 1
    faces = []
    coords = []
    lattice_id = {}
    # build each cube face as a grid; merge duplicate border vertices by
    # integer lattice coordinates
    ax_sets = [(0, 1, 2, 0), (0, 1, 2, n), (0, 2, 1, 0), (0, 2, 1, n),
               (1, 2, 0, 0), (1, 2, 0, n)]
    all_keys = []
    for (ua, va, wa, wval) in ax_sets:
        U, V = np.meshgrid(g, g, indexing="ij")
        L = np.zeros((side, side, 3), dtype=np.int64)
        L[..., ua] = U
        L[..., va] = V
        L[..., wa] = wval
        all_keys.append(L.reshape(-1, 3))
    keys = np.vstack(all_keys)
    flat = (keys[:, 0] * side + keys[:, 1]) * side + keys[:, 2]
    uniq, inv = np.unique(flat, return_inverse=True)
    lat = np.stack([uniq // (side * side), (uniq // side) % side, uniq % side], 1)
    p = lat.astype(float) / n * 2.0 - 1.0
    p /= np.linalg.norm(p, axis=1, keepdims=True)
    off = 0
    fl = []
    for fi, (ua, va, wa, wval) in enumerate(ax_sets):
        ids = inv[off:off + side * side].reshape(side, side)
        off += side * side
        i, j = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
        a = ids[i, j].ravel()
        b = ids[i + 1, j].ravel()
        c = ids[i + 1, j + 1].ravel()
        d = ids[i, j + 1].ravel()
        # orient outward: the face normal of (a, b, c) is +/- the w axis
        outward = (wval == n) == ((ua, va, wa) in ((0, 1, 2), (1, 2, 0)))
        if not outward:
            b, d = d, b
        tri = np.empty((2 * len(a), 3), dtype=np.int64)
        tri[0::2] = np.stack([a, b, c], 1)
        tri[1::2] = np.stack([a, c, d], 1)
        fl.append(tri)
    f = np.vstack(fl)
    x, y, z = p[:, 0], p[:, 1], p[:, 2]
    r = 1.0 + amplitude * (np.sin(9.0 * x + 0.4) * np.sin(7.0 * y + 1.1)
                           + 0.5 * np.sin(13.0 * z + 2.3) * np.cos(5.0 * x)) \
        + 0.1 * amplitude * rng.uniform(-1.0, 1.0, len(p)) / max(n / 64.0, 1.0)
    return normalize_edge_scale(p * r[:, None], f)


_GENERATORS = {
    "triangle": single_triangle,
    "square": square,
    "cube": cube,
    "tetrahedron": tetrahedron,
    "octahedron": octahedron,
    "pyramid": pyramid,
    "icosahedron": icosahedron,
}


def make(name: str, *args, **kwargs) -> SurfaceMesh:
    """Build a fixed solid by name (reference meshes.py:501)."""
    return build_half_edge_mesh(*_GENERATORS[name](*args, **kwargs))


def tiny_corpus() -> dict[str, SurfaceMesh]:
    """Meshes of at most 50 faces used against the brute-force oracle
    (reference meshes.py:507)."""
    out = {name: make(name) for name in
           ("triangle", "square", "cube", "tetrahedron", "octahedron",
            "pyramid", "icosahedron")}
    out["strip6"] = build_half_edge_mesh(*strip(6))
    out["grid4x4"] = build_half_edge_mesh(*grid(4, 4))
    out["saddle8"] = build_half_edge_mesh(*saddle_fan(8))
    out["saddle10"] = build_half_edge_mesh(*saddle_fan(10))
    out["torus4x6"] = build_half_edge_mesh(*torus(4, 6))
    return out


def bench_mesh(name: str) -> SurfaceMesh:
    """The named BASELINE.json configuration meshes."""
    if name == "icosphere20k":
        return build_half_edge_mesh(*normalize_edge_scale(*icosphere(5)))
    if name == "terrain1m":
        return build_half_edge_mesh(*terrain(708))
    if name == "knot4m":
        return build_half_edge_mesh(*torus_knot_tube())
    if name == "knot1m":  # configs[2] at a quarter of the size: the oracle's full-fan mode fits
        return build_half_edge_mesh(*torus_knot_tube(n_along=10000, n_around=50))
    if name == "knotg4m":  # configs[2] as stated: a high-genus (7) torus-knot tube, 4M faces
        return build_half_edge_mesh(*torus_knot_tube_handles())
    if name == "knotg1m":  # ... at a quarter of the size (full-fan oracle fits)
        return build_half_edge_mesh(*torus_knot_tube_handles(n_along=10000, n_around=50))
    if name == "sphere16m":
        return build_half_edge_mesh(*perturbed_sphere(1155))
    if name == "torus500k":
        return build_half_edge_mesh(*normalize_edge_scale(*bumpy_torus(500, 500)))
    raise KeyError(name)
