import sys, numpy as np
sys.path.insert(0, "/root/repo")
from paper_1305_1293_b200 import EngineConfig, run_pch
from paper_1305_1293_b200 import meshes as M
m = M.bench_mesh("knot4m")
eps = 1e-12
det, _ = run_pch(m, [0], EngineConfig(deterministic=True, epsilon_window=eps))
fd = np.isfinite(det)
for kw in ({}, {"fan_mode": "full_edges"}, {"recheck": False}, {"chain": 1}, {"k": 1024},
           {"fan_mode": "full_edges", "recheck": False}):
    d, st = run_pch(m, [0], EngineConfig(epsilon_window=eps, **kw))
    f = np.isfinite(d); both = f & fd
    r = (d[both] - det[both]) / np.maximum(det[both], 1e-12)
    idx = np.flatnonzero(both)[r > 1e-9]
    print(f"{kw}: longer {len(idx)} max {r.max():.2e} unreachable live {int((~f).sum())} det {int((~fd).sum())} "
          f"worst {idx[np.argsort(-(d[idx]-det[idx]))][:6].tolist()}", flush=True)
    if kw == {}:
        for v in idx[np.argsort(-(d[idx]-det[idx]))][:3]:
            he = np.flatnonzero(m.origin == v)
            nb = [int(m.origin[3*(h//3)+(h%3+1)%3]) for h in he]
            print(f"   v {int(v)} class {int(m.vertex_class[v])} det {det[v]:.6f} live {d[v]:.6f} "
                  f"nbrs det {[round(float(det[u]),4) for u in nb]} live {[round(float(d[u]),4) for u in nb]}", flush=True)
