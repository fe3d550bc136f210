"""One solve of a bench workload for ncu capture (development tool):
    python tools/prof_one.py WORKLOAD K [warmup]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1305_1293_b200 import EngineConfig, run_pch  # noqa: E402
from paper_1305_1293_b200 import meshes as M  # noqa: E402

name = sys.argv[1]
k = int(sys.argv[2])
warm = int(sys.argv[3]) if len(sys.argv) > 3 else 1
m = M.bench_mesh(name)
src = 354 * 709 + 354 if name == "terrain1m" else 0
for _ in range(warm + 1):
    d, st = run_pch(m, [src], EngineConfig(k=k))
print(st.time_kernel_ms, st.iterations, st.windows_propagated)
