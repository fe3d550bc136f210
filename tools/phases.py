"""Phase split (warp-cycle attribution) of single fields and batched rows.
    python tools/phases.py MESH [NROWS]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1305_1293_b200 import EngineConfig, meshes, run_pch, run_pch_rows  # noqa: E402

name = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 0
m = meshes.bench_mesh(name)
src = 354 * 709 + 354 if name == "terrain1m" else int(np.argmin(np.linalg.norm(m.positions - m.positions.mean(0), axis=1)))
cfg = EngineConfig(phase_times=True)
if n:
    srcs = np.random.default_rng(4096).choice(m.n_vertices, n, replace=False)
    run_pch_rows(m, srcs[:32], cfg)
    _, st = run_pch_rows(m, srcs, cfg)
else:
    run_pch(m, [src], cfg)
    _, st = run_pch(m, [src], cfg)
tot = st.time_select + st.time_propagate + st.time_compact + st.time_events
print(name, n or "single", f"kernel {st.time_kernel_ms:.2f} ms", {k: f"{getattr(st, k) / tot * 100:.1f}%" for k in
      ("time_select", "time_propagate", "time_compact", "time_events")}, "iters", st.iterations,
      "item_us", round(st.prop_item_us, 2), "stored", st.windows_stored, "propagated", st.windows_propagated)
