"""Large-configuration parity + timing on the GPU (development tool).

    python tools/bigcheck.py [knot4m] [sphere16m] [torus500k]

For each BASELINE.json configuration mesh: one single-source field from
the centre-most vertex, timed (best of 3, device events) and checked
against the sequential ICH oracle (checker only); for torus500k also a
batch of distance-matrix rows through run_pch_rows.
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def rel(a, b):
    fa, fb = np.isfinite(a), np.isfinite(b)
    if not np.array_equal(fa, fb):
        return float("inf")
    return float(np.max(np.abs(a[fa] - b[fa]) / np.maximum(np.abs(b[fa]), 1e-12)))


def main():
    from oracle import oracle as O
    from paper_1305_1293_b200 import EngineConfig, run_pch, run_pch_rows
    from paper_1305_1293_b200 import meshes as M
    names = sys.argv[1:] or ["knot4m", "sphere16m", "torus500k"]
    out = {}
    for name in names:
        t = time.time()
        m = M.bench_mesh(name)
        tb = time.time() - t
        src = int(np.argmin(np.linalg.norm(m.positions - m.positions.mean(0), axis=1)))
        if name == "knot4m":
            src = 0
        rec = {"faces": int(m.n_faces), "vertices": int(m.n_vertices), "build_s": round(tb, 1),
               "source": src}
        for k in (65536, 16384):  # the default (16384) last: its field is checked
            best = None
            for _ in range(3):
                d, st = run_pch(m, [src], EngineConfig(k=k))
                if best is None or st.time_kernel_ms < best[1].time_kernel_ms:
                    best = (d, st)
            d, st = best
            rec[f"k{k}"] = {"kernel_ms": round(st.time_kernel_ms, 3), "iters": st.iterations,
                            "propagated": st.windows_propagated,
                            "created": st.total_windows_created,
                            "regrows": st.buffer_regrows}
            print(name, k, rec[f"k{k}"], flush=True)
        t = time.time()
        ref, rs = O.run_ich(m, [src])
        rec["ich_s"] = round(time.time() - t, 2)
        rec["ich_windows"] = rs["total_windows_created"]
        rec["max_rel_err"] = rel(d, ref)
        rec["unreachable"] = int(np.sum(~np.isfinite(d)))
        rec["unreachable_ich"] = int(np.sum(~np.isfinite(ref)))
        both = np.isfinite(d) & np.isfinite(ref)
        rec["unreachable_both"] = int(np.sum(~np.isfinite(d) & ~np.isfinite(ref)))
        rec["max_rel_err_shared"] = float(np.max(np.abs(d[both] - ref[both]) /
                                                 np.maximum(np.abs(ref[both]), 1e-12)))
        print(name, "ich", rec["ich_s"], "s err", rec["max_rel_err"], flush=True)
        if name == "torus500k":
            rng = np.random.default_rng(4096)
            srcs = rng.choice(m.n_vertices, 64, replace=False)
            t = time.time()
            rows, st = run_pch_rows(m, srcs, EngineConfig(k=16384))
            dt = time.time() - t
            rec["rows64"] = {"wall_s": round(dt, 3), "sources_per_s": round(64 / dt, 2),
                             "kernel_ms_total": round(st.time_kernel_ms, 2)}
            errs = [rel(rows[i], O.run_ich(m, [int(srcs[i])])[0]) for i in range(2)]
            rec["rows64"]["max_rel_err_first2"] = max(errs)
            print(name, "rows", rec["rows64"], flush=True)
        out[name] = rec
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "bigcheck.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
