"""Generate golden vectors by running the REFERENCE package itself.

Run in the build container, where the reference is mounted read-only at
/root/reference (it never travels to the GPU box; the fixtures do):

    python tests/golden/make_golden.py

For every case the mesh (positions, faces), the sources, and the
reference's outputs are stored in ``tests/golden/<case>.npz``:
  ich_dist / ich_windows     -- pargeo.engine.run_ich   (engine.py:624)
  pch_dist / pch_windows     -- pargeo.engine.run_pch   (engine.py:433),
                                default EngineConfig(k=4096) with workers=4
  brute_dist (tiny meshes)   -- pargeo.oracle.brute_force_geodesic
                                (oracle.py:152), the exhaustive-unfolding
                                oracle, for meshes of at most 60 faces
Mesh generators are the reference's own (pargeo.meshes), so the fixtures
pin the exact inputs as well as the outputs.
"""
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))


def main():
    sys.path.insert(0, REF)
    from pargeo import meshes as R
    from pargeo.engine import EngineConfig, run_ich, run_pch
    from pargeo.mesh import build_half_edge_mesh
    from pargeo.oracle import brute_force_geodesic

    cases = []
    for name, m in R.tiny_corpus().items():
        for s in sorted({0, m.n_vertices // 2}):
            cases.append((f"tiny_{name}_s{s}", m.positions, m.faces, [s], True))
    for sub in (2, 3, 4, 5):
        p, f = R.normalize_edge_scale(*R.icosphere(sub))
        rng = np.random.default_rng(11)
        s = int(rng.integers(0, len(p)))
        cases.append((f"icosphere{20 * 4 ** sub}_s{s}", p, f, [s], False))
    p, f = R.normalize_edge_scale(*R.icosphere(4))
    cases.append(("icosphere5120_multi3", p, f, [0, 17, 101], False))
    cases.append(("icosphere5120_multi16",
                  p, f, sorted(np.random.default_rng(116).choice(len(p), 16, replace=False).tolist()), False))
    p, f = R.normalize_edge_scale(*R.bumpy_sphere(5))
    cases.append(("bumpy_sphere20k_s3", p, f, [3], False))
    p, f = R.normalize_edge_scale(*R.disk_patch(30))
    cases.append(("disk_patch_s0", p, f, [0], False))
    cases.append(("disk_patch_s2000", p, f, [2000], False))
    p, f = R.normalize_edge_scale(*R.bumpy_torus(60, 40))
    cases.append(("bumpy_torus4800_s5", p, f, [5], False))
    # noisy heightfield with a boundary: unreachable (shadowed) vertices
    rng = np.random.default_rng(1305)
    hts = rng.uniform(-0.35, 0.35, (41, 41))
    p, f = R.grid(40, 40, 1.0, lambda x, y: hts[x.astype(int), y.astype(int)]
                  + 0.8 * np.sin(0.3 * x) * np.cos(0.25 * y))
    p, f = R.normalize_edge_scale(p, f)
    cases.append(("terrain3200_center", p, f, [20 * 41 + 20], False))
    cases.append(("terrain3200_corner", p, f, [0], False))

    for name, p, f, src, tiny in cases:
        m = build_half_edge_mesh(p, f)
        di, si = run_ich(m, src)
        dp, sp = run_pch(m, src, EngineConfig(k=4096, workers=4))
        rec = dict(positions=np.asarray(p, np.float64), faces=np.asarray(f, np.int64),
                   sources=np.asarray(src, np.int64), ich_dist=di,
                   ich_windows=np.int64(si.total_windows_created),
                   ich_propagated=np.int64(si.windows_propagated),
                   pch_dist=dp, pch_windows=np.int64(sp.total_windows_created))
        if tiny:
            rec["brute_dist"] = brute_force_geodesic(m, src[0])
        np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **rec)
        print(f"{name}: F={m.n_faces} ich_windows={si.total_windows_created} "
              f"unreachable={int(np.sum(~np.isfinite(di)))}", flush=True)


if __name__ == "__main__":
    main()
