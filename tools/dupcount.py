"""Duplicate fan windows dropped per field (development check).
    python tools/dupcount.py MESH..."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1305_1293_b200 import EngineConfig, meshes, run_pch  # noqa: E402

for name in sys.argv[1:]:
    m = meshes.bench_mesh(name)
    src = 354 * 709 + 354 if name == "terrain1m" else int(np.argmin(np.linalg.norm(m.positions - m.positions.mean(0), axis=1)))
    for dd in (True, False):
        for det in (False, True):
            if det and name in ("knot4m", "sphere16m"):
                continue
            d, st = run_pch(m, [src], EngineConfig(dedupe=dd, deterministic=det))
            print(name, "dedupe" if dd else "keep  ", "det " if det else "live", "created", st.total_windows_created,
                  "dup", st.pruned_duplicate, "fans", st.fans_emitted, f"{st.time_kernel_ms:.2f} ms", flush=True)
