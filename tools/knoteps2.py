"""knot4m: live vs deterministic solver per epsilon_window / fan mode
(development tool): vertices where the live field is longer, holes."""
import sys
import numpy as np
sys.path.insert(0, "/root/repo")
from paper_1305_1293_b200 import EngineConfig, run_pch
from paper_1305_1293_b200 import meshes as M
m = M.bench_mesh("knot4m")
for eps in (1e-6, 1e-12):
    det, _ = run_pch(m, [0], EngineConfig(deterministic=True, epsilon_window=eps))
    fd = np.isfinite(det)
    for kw in ({}, {"fan_mode": "full_edges"}):
        d, st = run_pch(m, [0], EngineConfig(epsilon_window=eps, **kw))
        f = np.isfinite(d); both = f & fd
        r = (d[both] - det[both]) / np.maximum(det[both], 1e-12)
        idx = np.flatnonzero(both)[r > 1e-9]
        print(f"eps {eps:g} {kw}: {st.time_kernel_ms:.0f} ms live longer {len(idx)} (max {r.max():.2e}) "
              f"shorter {int((r < -1e-9).sum())} (min {r.min():.2e}) unreachable live {int((~f).sum())} "
              f"det {int((~fd).sum())} worst {idx[np.argsort(-(d[idx]-det[idx]))][:4].tolist()}", flush=True)
