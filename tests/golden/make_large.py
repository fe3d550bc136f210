"""Oracle fixtures for the BASELINE.json configuration meshes (configs[1-4]).

    python tests/golden/make_large.py [case ...]        # all cases by default

TEST INFRASTRUCTURE.  The sequential ICH restatement in oracle/ (reference
pkg/src/pargeo/engine.py:624 run_ich; pinned window-for-window against the
reference itself by tests/test_oracle_golden.py) takes 3 s to 11 min per
field on these meshes, far too long for the GPU suite, so it runs once
here and the fixtures are committed:

  large_<case>.npz
    mesh       workload name (paper_1305_1293_b200.meshes.bench_mesh)
    mesh_sig   (n_vertices, n_faces, sum of half-edge lengths): detects a
               generator change that would invalidate the fixture
    source     the source vertex
    holes      every vertex the oracle leaves at +inf (int32, complete)
    idx, val   a seeded sample of 32768 vertices (16384 for rows) and their
               oracle distances
    n_finite, finite_sum   count and sum of the finite distances
    windows    oracle windows created (ICH)
    holes_full, val_full, windows_full
               the same with the reference's fan_mode="full_edges" (every
               saddle wedge emitted un-clipped, EngineConfig.fan_mode,
               reference engine.py:57): no thin-fan rounding holes, the
               field the default mode approximates where it has holes

The full fields go to scratch/ (git-ignored) for development diagnostics.
"""
from __future__ import annotations

import multiprocessing as mp
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

TERRAIN_SRC = 354 * 709 + 354
# configs[4] rows: the first ten sources of the bench's seeded draw on the
# 500k-face torus (rows 1 and 2 are the ones with rounding holes)
TORUS_ROW_SOURCES = [102311, 246971, 207580, 114359, 174139, 190541, 200393, 2108, 151566, 24267]


def centre_source(m):
    return int(np.argmin(np.linalg.norm(m.positions - m.positions.mean(0), axis=1)))


def cases():
    out = [("terrain1m", "terrain1m", "terrain"),
           ("torus500k", "torus500k", "centre"),
           ("sphere16m", "sphere16m", "centre"),
           ("knot4m", "knot4m", 0),
           ("knot1m", "knot1m", 0),
           ("knotg1m", "knotg1m", 0),
           ("knotg4m", "knotg4m", 0)]
    out += [(f"torus500k_row{i}", "torus500k", s) for i, s in enumerate(TORUS_ROW_SOURCES)]
    return out


def mesh_sig(m):
    return np.array([m.n_vertices, m.n_faces, float(np.sum(m.length))], np.float64)


def make(case):
    from oracle import oracle as O
    from paper_1305_1293_b200 import meshes as M
    name, mesh, src = case
    m = M.bench_mesh(mesh)
    if src == "terrain":
        src = TERRAIN_SRC
    elif src == "centre":
        src = centre_source(m)
    t = time.time()
    cached = os.path.join(ROOT, "scratch", f"ich_{name}.npy")
    if os.path.exists(cached) and os.environ.get("REUSE_CLIP"):
        d, st = np.load(cached), None
    else:
        d, st = O.run_ich(m, [src])
    if os.environ.get("NO_FULL"):
        dfull, stf = None, None
    else:
        dfull, stf = O.run_ich(m, [src], fan_mode="full_edges")
    dt = time.time() - t
    nsamp = 16384 if "_row" in name else 32768
    rng = np.random.default_rng(20260)
    idx = np.sort(rng.choice(m.n_vertices, min(nsamp, m.n_vertices), replace=False)).astype(np.int32)
    fin = np.isfinite(d)
    old = os.path.join(HERE, f"large_{name}.npz")
    windows = (st["total_windows_created"] if st else int(np.load(old)["windows"]))
    rec = dict(mesh=np.array(mesh), mesh_sig=mesh_sig(m), source=np.int64(src),
               holes=np.flatnonzero(~fin).astype(np.int32), idx=idx, val=d[idx],
               n_finite=np.int64(fin.sum()), finite_sum=np.float64(np.sum(d[fin])),
               windows=np.int64(windows))
    if dfull is not None:
        rec.update(holes_full=np.flatnonzero(~np.isfinite(dfull)).astype(np.int32),
                   val_full=dfull[idx], windows_full=np.int64(stf["total_windows_created"]))
    np.savez_compressed(os.path.join(HERE, f"large_{name}.npz"), **rec)
    os.makedirs(os.path.join(ROOT, "scratch"), exist_ok=True)
    np.save(os.path.join(ROOT, "scratch", f"ich_{name}.npy"), d)
    if dfull is None:
        return f"{name}: src={src} V={m.n_vertices} holes={int((~fin).sum())} windows={windows} (no full-fan oracle)"
    np.save(os.path.join(ROOT, "scratch", f"ichfull_{name}.npy"), dfull)
    return (f"{name}: src={src} V={m.n_vertices} holes={int((~fin).sum())} "
            f"holes_full={int((~np.isfinite(dfull)).sum())} windows={windows} "
            f"full={stf['total_windows_created']} ich {dt:.1f}s")


def main():
    want = set(sys.argv[1:])
    todo = [c for c in cases() if not want or c[0] in want]
    # longest first; at most 6 at once (the 16M-face mesh needs ~10 GB)
    order = {"knot4m": 0, "sphere16m": 1}
    todo.sort(key=lambda c: order.get(c[0], 2))
    with mp.get_context("spawn").Pool(min(6, len(todo))) as pool:
        for line in pool.imap_unordered(make, todo):
            print(line, flush=True)


if __name__ == "__main__":
    main()
