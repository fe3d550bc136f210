"""Live solver vs the deterministic (frozen-table) solver on stress meshes
(development tool): vertices where the live field is longer than the
deterministic one by more than 1e-9 relative, and reachability flags.

    python tools/livecheck.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1305_1293_b200 import EngineConfig, build_half_edge_mesh, run_pch  # noqa: E402
from paper_1305_1293_b200 import meshes as M  # noqa: E402

cases = []
for na in (1000, 2000, 5000):
    cases.append((f"knot_{na}x100", build_half_edge_mesh(*M.torus_knot_tube(n_along=na)), [0, 7]))
cases.append(("torus500k", M.bench_mesh("torus500k"), [246971, 207580]))
for name, m, srcs in cases:
    for s in srcs:
        det, _ = run_pch(m, [s], EngineConfig(deterministic=True))
        fd = np.isfinite(det)
        for chain in (1, 2, 3):
            for rep in range(2):
                d, st = run_pch(m, [s], EngineConfig(chain=chain))
                f = np.isfinite(d)
                both = f & fd
                r = (d[both] - det[both]) / np.maximum(det[both], 1e-12)
                bad = np.flatnonzero(both)[r > 1e-9]
                print(f"{name} src {s} chain {chain}: longer {len(bad)} max {r.max():.2e} "
                      f"shorter {int((r < -1e-9).sum())} live-only-reach {int((f & ~fd).sum())} "
                      f"det-only-reach {int((~f & fd).sum())} worst {bad[np.argsort(-r[r > 1e-9])][:4].tolist()}",
                      flush=True)
