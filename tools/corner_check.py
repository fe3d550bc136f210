"""terrain3200_corner against its golden rule, repeated (development tool)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from conftest import TOL, load_golden, max_rel_dev
from paper_1305_1293_b200 import EngineConfig, run_pch
m, g = load_golden("terrain3200_corner")
ich, pch = g["ich_dist"], g["pch_dist"]
mask = np.isfinite(ich) & np.isfinite(pch)
agree = mask & (np.abs(ich - pch) <= TOL * np.maximum(np.abs(ich), 1e-12))
lo, hi = np.minimum(ich, pch), np.maximum(ich, pch)
split = mask & ~agree
res = []
for k in (1, 64, 4096, 65536):
    for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
        d, st = run_pch(m, g["sources"], EngineConfig(k=k))
        a = bool(np.all(np.isfinite(d[mask])))
        e = max_rel_dev(d[agree], ich[agree])
        below = int(np.sum(d[split] < lo[split] * (1 - TOL)))
        above = int(np.sum(d[split] > hi[split] * (1 + TOL)))
        bad = np.flatnonzero(agree & (np.abs(d - ich) > TOL * np.maximum(np.abs(ich), 1e-12)))
        ok = a and e <= TOL and below == 0 and above == 0
        res.append(ok)
        if not ok:
            print(f"k={k} rep={rep} FAIL reach={a} err_agree={e:.3e} n_bad={len(bad)} below={below} above={above} "
                  f"bad={bad[:5].tolist()} d={d[bad[:3]].tolist()} ich={ich[bad[:3]].tolist()} pch={pch[bad[:3]].tolist()}")
print(os.environ.get("PCH_B200_LIB", "in-tree"), f"{sum(res)}/{len(res)} ok")
