import sys, numpy as np
sys.path.insert(0, "/root/repo")
from paper_1305_1293_b200 import EngineConfig, run_pch
from paper_1305_1293_b200 import meshes as M
m = M.bench_mesh("knot4m")
for eps in (1e-6, 1e-9, 1e-12):
    det, _ = run_pch(m, [0], EngineConfig(deterministic=True, epsilon_window=eps))
    fd = np.isfinite(det)
    for chain in (3,):
        d, st = run_pch(m, [0], EngineConfig(chain=chain, epsilon_window=eps))
        f = np.isfinite(d); both = f & fd
        r = (d[both] - det[both]) / np.maximum(det[both], 1e-12)
        print(f"eps {eps:g}: det unreachable {int((~fd).sum())} live unreachable {int((~f).sum())} "
              f"live longer {int((r > 1e-9).sum())} (max {r.max():.2e}) shorter {int((r < -1e-9).sum())} (min {r.min():.2e}) "
              f"live ms {st.time_kernel_ms:.0f} windows {st.total_windows_created}", flush=True)
    if eps == 1e-6:
        base = det
    else:
        b = np.isfinite(base) & fd
        rr = (det[b] - base[b]) / np.maximum(base[b], 1e-12)
        print(f"   det(eps) vs det(1e-6): longer {int((rr > 1e-9).sum())} shorter {int((rr < -1e-9).sum())} min {rr.min():.2e}", flush=True)
