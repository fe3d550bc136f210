"""Golden SurfaceMesh arrays built by the REFERENCE (pargeo.mesh.
build_half_edge_mesh, mesh.py:142) for a few meshes with boundaries,
saddles and noise; run here where /root/reference is mounted:

    python tests/golden/make_mesh_golden.py

tests/test_mesh.py checks the native builder against them bit for bit."""
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "mesh_arrays.npz")


def main():
    sys.path.insert(0, REF)
    from pargeo import meshes as R
    from pargeo.mesh import build_half_edge_mesh
    rng = np.random.default_rng(0)
    p, f = R.grid(20, 20)
    cases = {"icosphere5120": R.normalize_edge_scale(*R.icosphere(4)),
             "bumpy_torus4800": R.normalize_edge_scale(*R.bumpy_torus(60, 40)),
             "disk_patch": R.normalize_edge_scale(*R.disk_patch(12)),
             "saddle10": R.saddle_fan(10),
             "noisy_grid": (p + rng.normal(0, 0.1, p.shape), f)}
    rec = {}
    for name, (p, f) in cases.items():
        m = build_half_edge_mesh(p, f)
        rec[f"{name}/positions"] = np.asarray(p, np.float64)
        rec[f"{name}/faces"] = np.asarray(f, np.int64)
        for k in ("origin", "opposite", "length", "corner_angle", "total_angle", "vertex_class",
                  "outgoing", "on_boundary"):
            rec[f"{name}/{k}"] = getattr(m, k)
    np.savez_compressed(OUT, **rec)
    print(OUT, sorted({k.split("/")[0] for k in rec}))


if __name__ == "__main__":
    main()
