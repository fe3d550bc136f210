"""Batched distance-matrix rows throughput (development tool).

    python tools/rowsbench.py MESH NSRC [SPEC ...]

SPEC = R or "R=32,k=65536,chain=1,dmin=0.4" (batch size PCH_ROWS, engine
config, controller floor PCH_DELTA_MIN in mean edges).  Times
pch_run_rows over NSRC random sources for each spec and checks two rows
against the sequential ICH oracle."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from oracle import oracle as O  # noqa: E402
from paper_1305_1293_b200 import EngineConfig, run_pch_rows  # noqa: E402
from paper_1305_1293_b200 import meshes as M  # noqa: E402

name, n = sys.argv[1], int(sys.argv[2])
specs = sys.argv[3:] or ["1", "8", "32"]
m = M.bench_mesh(name)
src = np.random.default_rng(4096).choice(m.n_vertices, n, replace=False)
refs = {i: O.run_ich(m, [int(src[i])])[0] for i in (0, n - 1)}
for spec in specs:
    kv = dict(x.split("=") for x in spec.split(",")) if "=" in spec else {"R": spec}
    R = int(kv.pop("R", 32))
    os.environ["PCH_ROWS"] = str(R)
    os.environ.pop("PCH_DELTA_MIN", None)
    if "dmin" in kv:
        os.environ["PCH_DELTA_MIN"] = kv.pop("dmin")
    cfg = EngineConfig(**{k: int(v) for k, v in kv.items()})
    run_pch_rows(m, src[: min(n, R)], cfg)  # warm / allocate
    t = time.perf_counter()
    rows, st = run_pch_rows(m, src, cfg)
    dt = time.perf_counter() - t
    errs = []
    for i, ref in refs.items():
        fin = np.isfinite(ref)
        same = np.array_equal(np.isfinite(rows[i]), fin)
        errs.append(float(np.max(np.abs(rows[i][fin] - ref[fin]) / np.maximum(ref[fin], 1e-12))) if same else np.inf)
    print(f"{name} {spec:34s} sources={n} wall={dt:.3f}s sources/s={n / dt:.1f} kernel_ms={st.time_kernel_ms:.1f} "
          f"iters={st.iterations} windows={st.total_windows_created} regrows={st.buffer_regrows} "
          f"err={max(errs):.2e}", flush=True)
