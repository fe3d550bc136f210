"""Solve a bench mesh and report self-consistency (development check):
    python tools/meshprobe.py MESH [variant ...]   (variants as in fieldcheck)"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1305_1293_b200 import EngineConfig, meshes, run_pch  # noqa: E402
from tools.fieldcheck import parse  # noqa: E402

m = meshes.bench_mesh(sys.argv[1])
u = m.origin
v = m.origin[3 * (np.arange(len(u)) // 3) + (np.arange(len(u)) + 1) % 3]
for var in sys.argv[2:] or ["base"]:
    d, st = run_pch(m, [0], EngineConfig(**parse(var)))
    fin = np.isfinite(d)
    both = fin[u] & fin[v]
    gap = np.abs(d[u] - d[v]) - m.length * (1 + 1e-12)
    lip = int(np.unique(np.concatenate([u[both & (gap > 1e-9 * d[fin].max())], v[both & (gap > 1e-9 * d[fin].max())]])).size)
    print(sys.argv[1], var, json.dumps({"faces": int(m.n_faces), "holes": int((~fin).sum()), "lipschitz_vertices": lip,
                                        "max_dist": float(d[fin].max()), "kernel_ms": round(st.time_kernel_ms, 1),
                                        "windows": st.total_windows_created, "iters": st.iterations}), flush=True)
