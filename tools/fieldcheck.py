"""Full-field comparison of GPU solver variants against an oracle field
(development diagnostic; the committed test is tests/test_gpu_large.py).

    python tools/fieldcheck.py CASE [variant ...]

CASE names a fixture of tests/golden/make_large.py; the oracle's full
field is read from scratch_gpu/ich_CASE.npy (copied there from scratch/
so it travels to the GPU box).  A variant is a comma-separated list of
EngineConfig overrides, e.g. ``deterministic=1``, ``chain=1,recheck=0``,
``epsilon_window=1e-12``; ``base`` is the default configuration.
Reports, per variant: holes (GPU / oracle / GPU-only), vertices longer or
shorter than the oracle by more than 1e-9 relative, the worst relative
error on vertices both reach, kernel ms.
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def parse(v):
    kw = {}
    if v == "base":
        return kw
    for item in v.split(","):
        k, x = item.split("=")
        if k in ("deterministic", "recheck"):
            kw[k] = bool(int(x))
        elif k in ("chain", "k", "pool_capacity"):
            kw[k] = int(x)
        elif k in ("fan_mode", "tiny_rule"):
            kw[k] = x
        else:
            kw[k] = float(x)
    return kw


def compare(d, ref):
    fd, fr = np.isfinite(d), np.isfinite(ref)
    both = fd & fr
    rel = (d[both] - ref[both]) / np.maximum(ref[both], 1e-12)
    idx = np.flatnonzero(both)
    long_ = idx[rel > 1e-9]
    short = idx[rel < -1e-9]
    return {"holes_gpu": int((~fd).sum()), "holes_ref": int((~fr).sum()),
            "gpu_only_holes": int((~fd & fr).sum()), "filled": int((fd & ~fr).sum()),
            "long": int(len(long_)), "short": int(len(short)),
            "max_abs_rel": float(np.abs(rel).max()) if rel.size else 0.0,
            "long_ids": long_[:20].tolist(), "short_ids": short[:20].tolist(),
            "gpu_only_ids": np.flatnonzero(~fd & fr)[:20].tolist()}


def rows_main(cases, variants):
    """--rows CASE... : one run_pch_rows over the cases' sources (same mesh)."""
    from paper_1305_1293_b200 import EngineConfig, meshes, run_pch_rows
    gs = [dict(np.load(os.path.join(ROOT, "tests", "golden", f"large_{c}.npz"))) for c in cases]
    m = meshes.bench_mesh(str(gs[0]["mesh"]))
    src = [int(g["source"]) for g in gs]
    for v in variants:
        rows, st = run_pch_rows(m, src, EngineConfig(**parse(v)))
        for c, r in zip(cases, rows):
            ref = np.load(os.path.join(ROOT, "scratch_gpu", f"ich_{c}.npy"))
            rep = compare(r, ref)
            print("rows", c, v, json.dumps(rep), flush=True)
        if os.environ.get("FIELDCHECK_SAVE"):
            np.save(os.path.join(ROOT, "gpurun_out", f"rows_{v.replace(',', '_').replace('=', '')}.npy"), rows)


def main():
    from paper_1305_1293_b200 import EngineConfig, meshes, run_pch
    if sys.argv[1] == "--rows":
        cases = [a for a in sys.argv[2:] if "=" not in a and a != "base"]
        variants = [a for a in sys.argv[2:] if "=" in a or a == "base"] or ["base"]
        return rows_main(cases, variants)
    case = sys.argv[1]
    variants = sys.argv[2:] or ["base"]
    g = dict(np.load(os.path.join(ROOT, "tests", "golden", f"large_{case}.npz")))
    # FIELDCHECK_REF=ichfull compares against the full-fan oracle field
    ref = np.load(os.path.join(ROOT, "scratch_gpu", f"{os.environ.get('FIELDCHECK_REF', 'ich')}_{case}.npy"))
    m = meshes.bench_mesh(str(g["mesh"]))
    src = int(g["source"])
    out = {}
    for v in variants:
        d, st = run_pch(m, [src], EngineConfig(**parse(v)))
        rep = compare(d, ref)
        rep["kernel_ms"] = round(st.time_kernel_ms, 2)
        rep["windows"] = st.total_windows_created
        out[v] = rep
        print(case, v, json.dumps(rep), flush=True)
        if os.environ.get("FIELDCHECK_SAVE"):
            np.save(os.path.join(ROOT, "gpurun_out", f"field_{case}_{v.replace(',', '_').replace('=', '')}.npy"), d)
    with open(os.path.join(ROOT, "gpurun_out", f"fieldcheck_{case}.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
