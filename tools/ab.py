"""A/B timing of library builds (development tool).

    python tools/ab.py WORKLOAD LIB1 [LIB2 ...] [--cfg k=v,...] [--reps N]

Each LIB (a built libpch_b200.so) runs in its own process (PCH_B200_LIB),
N interleaved rounds of 5 solves; prints the median kernel ms per build.
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import os, sys, json, numpy as np
sys.path.insert(0, os.environ["ROOT"])
from paper_1305_1293_b200 import EngineConfig, run_pch
from paper_1305_1293_b200 import meshes as M
name = os.environ["WL"]
m = M.bench_mesh(name)
src = 354 * 709 + 354 if name == "terrain1m" else int(np.argmin(np.linalg.norm(m.positions - m.positions.mean(0), axis=1)))
kw = json.loads(os.environ.get("CFG", "{}"))
nrows = int(kw.pop("rows", 0))
cfg = EngineConfig(**kw)
if nrows:
    from paper_1305_1293_b200 import run_pch_rows
    srcs = np.random.default_rng(4096).choice(m.n_vertices, nrows, replace=False)
    run_pch_rows(m, srcs[:32], cfg)
    ts = []
    for _ in range(int(os.environ.get("N", "2"))):
        rows, st = run_pch_rows(m, srcs, cfg)
        ts.append(st.time_kernel_ms / nrows)  # ms per row
else:
  for _ in range(3):
    run_pch(m, [src], cfg)
  ts = []
  for _ in range(int(os.environ.get("N", "5"))):
    d, st = run_pch(m, [src], cfg)
    ts.append(st.time_kernel_ms)
print(json.dumps({"ms": ts, "iters": st.iterations, "created": st.total_windows_created}))
'''


def main():
    args = sys.argv[1:]
    wl = args[0]
    cfg, reps, libs = {}, 3, []
    i = 1
    while i < len(args):
        if args[i] == "--cfg":
            for kv in args[i + 1].split(","):
                k, v = kv.split("=")
                cfg[k] = int(v) if v.isdigit() else (float(v) if v.replace(".", "").replace("e-", "").isdigit() else v)
            i += 2
        elif args[i] == "--reps":
            reps = int(args[i + 1])
            i += 2
        else:
            libs.append(args[i])
            i += 1
    res = {lib: [] for lib in libs}
    info = {}
    for _ in range(reps):
        for lib in libs:
            env = dict(os.environ, ROOT=ROOT, WL=wl, CFG=json.dumps(cfg), PCH_B200_LIB=os.path.abspath(lib))
            out = subprocess.run([sys.executable, "-c", CHILD], capture_output=True, text=True, env=env)
            if out.returncode:
                print(lib, out.stderr[-800:])
                continue
            r = json.loads(out.stdout.strip().splitlines()[-1])
            res[lib] += r["ms"]
            info[lib] = (r["iters"], r["created"])
    for lib in libs:
        ts = sorted(res[lib])
        if ts:
            print(f"{wl} {os.path.basename(os.path.dirname(lib)) or lib}/{os.path.basename(lib)}: "
                  f"median {ts[len(ts) // 2]:.3f} ms min {ts[0]:.3f} (n={len(ts)}) iters/created {info.get(lib)}")


if __name__ == "__main__":
    main()
