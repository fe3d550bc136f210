"""Per-row flag / error check of batched rows against single fields and
the ICH oracle (development tool).

    python tools/rowscheck.py MESH NSRC
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402
from paper_1305_1293_b200 import run_pch, run_pch_rows  # noqa: E402
from paper_1305_1293_b200 import meshes as M  # noqa: E402

name, n = sys.argv[1], int(sys.argv[2])
m = M.bench_mesh(name)
src = np.random.default_rng(4096).choice(m.n_vertices, 64, replace=False)[:n]
rows, _ = run_pch_rows(m, src)
for i, s in enumerate(src):
    ref, _ = O.run_ich(m, [int(s)])
    one, _ = run_pch(m, [int(s)])
    fr, fo, fi = np.isfinite(rows[i]), np.isfinite(one), np.isfinite(ref)
    both = fr & fi
    err = float(np.max(np.abs(rows[i][both] - ref[both]) / np.maximum(ref[both], 1e-12)))
    print(f"row {i} src {int(s)}: unreachable rows={int((~fr).sum())} single={int((~fo).sum())} "
          f"ich={int((~fi).sum())} rows-only={np.flatnonzero(~fr & fi)[:8].tolist()} "
          f"ich-only={np.flatnonzero(fr & ~fi)[:8].tolist()} err_shared={err:.2e}", flush=True)
