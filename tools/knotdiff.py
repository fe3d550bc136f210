"""knot4m: where the GPU field and the ICH oracle disagree (development tool).

    python tools/knotdiff.py
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402
from paper_1305_1293_b200 import EngineConfig, run_pch  # noqa: E402
from paper_1305_1293_b200 import meshes as M  # noqa: E402

m = M.bench_mesh("knot4m")
t = time.time()
ref, _ = O.run_ich(m, [0])
print(f"ich {time.time() - t:.0f}s unreachable {int((~np.isfinite(ref)).sum())}", flush=True)
fi = np.isfinite(ref)
for kw in ({"chain": 2}, {"chain": 3}, {"chain": 3, "deterministic": True}, {"chain": 1}):
    d, st = run_pch(m, [0], EngineConfig(**kw))
    fd = np.isfinite(d)
    both = fd & fi
    r = (d[both] - ref[both]) / np.maximum(ref[both], 1e-12)
    big = np.abs(r) > 1e-9
    print(f"{kw}: {st.time_kernel_ms:.0f} ms unreachable {int((~fd).sum())} both-unreach "
          f"{int((~fd & ~fi).sum())} ours-only-reach {int((fd & ~fi).sum())} ich-only-reach "
          f"{int((~fd & fi).sum())} | shared {int(both.sum())}: |rel|>1e-9 at {int(big.sum())} "
          f"(ours longer {int((r > 1e-9).sum())}, max {r.max():.2e}; ours shorter "
          f"{int((r < -1e-9).sum())}, min {r.min():.2e})", flush=True)
    if big.any():
        idx = np.flatnonzero(both)[np.argsort(-np.abs(r))[:5]]
        print("   worst vertices", idx.tolist(), "ours", d[idx].round(4).tolist(), "ich",
              ref[idx].round(4).tolist(), flush=True)
