"""GPU vs oracle on torus-knot tubes of growing length (development tool)."""
import sys
import time

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from oracle import oracle as O  # noqa: E402
from paper_1305_1293_b200 import EngineConfig, run_pch  # noqa: E402
from paper_1305_1293_b200 import meshes as M  # noqa: E402
from paper_1305_1293_b200.mesh import build_half_edge_mesh  # noqa: E402

for na in [int(x) for x in sys.argv[1:]] or [400, 1000, 5000]:
    m = build_half_edge_mesh(*M.torus_knot_tube(n_along=na, n_around=100))
    for k in (16384, 65536):
        for det in (False, True):
            d, st = run_pch(m, [0], EngineConfig(k=k, deterministic=det))
            print(na, m.n_faces, k, det, "unreach", int(np.sum(~np.isfinite(d))), "iters", st.iterations,
                  "ms", round(st.time_kernel_ms, 2), "created", st.total_windows_created,
                  "regrow", st.buffer_regrows, flush=True)
    if na <= 5000:
        t = time.time()
        ref, rs = O.run_ich(m, [0])
        fin = np.isfinite(ref)
        same = np.array_equal(np.isfinite(d), fin)
        err = float(np.max(np.abs(d[fin] - ref[fin]) / np.maximum(ref[fin], 1e-12))) if same else None
        bad = np.where(np.isfinite(d) != fin)[0][:10]
        print(na, "ich unreach", int(np.sum(~fin)), "err", err, "first mismatches", bad.tolist(),
              round(time.time() - t, 1), "s", flush=True)
