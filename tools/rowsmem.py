"""Batched rows on the 16M-face sphere: the batch size adapts to device
memory instead of failing (development tool)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1305_1293_b200 import run_pch, run_pch_rows  # noqa: E402
from paper_1305_1293_b200 import meshes as M  # noqa: E402

m = M.bench_mesh("sphere16m")
src = np.random.default_rng(7).choice(m.n_vertices, 8, replace=False)
t = time.perf_counter()
rows, st = run_pch_rows(m, src)
dt = time.perf_counter() - t
one, _ = run_pch(m, [int(src[3])])
fin = np.isfinite(one)
err = float(np.max(np.abs(rows[3][fin] - one[fin]) / np.maximum(one[fin], 1e-12)))
print(f"sphere16m rows: 8 sources in {dt:.2f}s ({8 / dt:.1f}/s), iters {st.iterations}, "
      f"flags equal {np.array_equal(np.isfinite(rows[3]), fin)}, max rel vs single {err:.2e}", flush=True)
