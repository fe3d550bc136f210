"""Per-iteration timeline of one traced solve, split into iterations that
end with a grid barrier and CTA-local ones (development tool).

    PCH_B200_LIB=altlib/dev/libpch_b200.so python tools/trace_split.py WORKLOAD

(the library built with tools/build_variant.sh dev -DPCH_DEVTOOLS: the
default build carries no trace instrumentation)
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from tools.sweep import TR  # noqa: E402


def main():
    from paper_1305_1293_b200 import EngineConfig, run_pch
    from paper_1305_1293_b200 import meshes as M
    name = sys.argv[1]
    m = M.bench_mesh(name)
    src = 354 * 709 + 354 if name == "terrain1m" else int(np.argmin(np.linalg.norm(m.positions - m.positions.mean(0), axis=1)))
    for _ in range(2):
        run_pch(m, [src], EngineConfig())
    os.environ["PCH_TRACE"] = "/tmp/pch_trace.bin"
    d, st = run_pch(m, [src], EngineConfig())
    a = np.fromfile("/tmp/pch_trace.bin", dtype=np.uint64).reshape(-1, len(TR)).astype(np.float64)
    a = a[a[:, 0] > 0]
    col = {k: i for i, k in enumerate(TR)}
    t0 = a[:, col["t0"]]
    dur = np.diff(t0) / 1e3
    a = a[:-1]
    t0 = t0[:-1]
    glob = a[:, col["b1"]] > 0
    print(f"{name}: {st.time_kernel_ms:.2f} ms (traced), {len(a) + 1} iterations, {int(glob.sum())} global")
    for lab, msk in (("global", glob), ("local", ~glob)):
        if not msk.any():
            continue
        def rel(k):
            v = a[msk, col[k]]
            ok = v > 0
            return np.mean(v[ok] - t0[msk][ok]) / 1e3 if ok.any() else float("nan")
        print(f"  {lab:6s} n={int(msk.sum()):4d} mean dur {dur[msk].mean():6.2f} us (sum {dur[msk].sum()/1e3:.2f} ms)"
              f" | from t0: start_max {rel('start_max'):5.2f} trip0 {rel('trip0'):5.2f} loaded {rel('loaded'):5.2f}"
              f" work_end {rel('work_end'):5.2f} routed {rel('routed'):5.2f} scan_end {rel('scan_end'):5.2f}"
              f" a_end {rel('a_end'):5.2f} | nS {a[msk, col['ns']].mean():.0f}")


if __name__ == "__main__":
    main()
