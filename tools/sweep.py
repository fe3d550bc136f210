"""Parameter sweep of the GPU engine on a bench mesh (development tool).

    python tools/sweep.py WORKLOAD "k=65536,chain=3;k=16384,dmin=0.4" [--trace] [--nocheck]

(dmin / delta set the PCH_DELTA_MIN / PCH_DELTA development overrides:
controller step floor / fixed step, in mean edge lengths.)

Each configuration is run 3 times (best device time reported) and checked
against the sequential ICH oracle (test infrastructure, checker only).
With --trace (needs a -DPCH_DEVTOOLS build, PCH_B200_LIB=altlib/dev/...),
PCH_TRACE is set and the per-iteration timeline of the last
run is summarised (phase A / barrier / phase B shares).
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

TR = ("t0", "a_end", "b1", "b_end", "b2", "ns", "np", "nc", "nf", "ntv", "tsel", "fan_end",
      "start_max", "work_end", "scan_end", "trip0", "loaded", "routed")


def parse(spec):
    out = {}
    for kv in spec.split(","):
        if not kv:
            continue
        k, v = kv.split("=")
        out[k] = float(v) if "." in v else int(v)
    env = {}
    for key, var in (("dmin", "PCH_DELTA_MIN"), ("delta", "PCH_DELTA"), ("dmax", "PCH_DELTA_MAX"), ("tpb", "PCH_TPB")):
        if key in out:
            env[var] = str(out.pop(key))
    out["_env"] = env
    for b in ("deterministic", "recheck"):
        if b in out:
            out[b] = bool(out[b])
    return out


def trace_summary(path):
    a = np.fromfile(path, dtype=np.uint64).reshape(-1, len(TR)).astype(np.float64)
    a = a[a[:, 0] > 0]
    t0, ae, b1, be, b2 = (a[:, i] for i in range(5))
    tot = (b2[-1] - t0[0]) / 1e3
    ph_a = np.sum(ae - t0) / 1e3
    bar1 = np.sum(b1 - ae) / 1e3
    ph_b = np.sum(be - b1) / 1e3
    bar2 = np.sum(b2 - be) / 1e3
    ns = a[:, 5]
    fan = np.sum(np.maximum(a[:, 11] - b1, 0)) / 1e3
    print(f"   trace: iters={len(a)} total={tot:.0f}us A={ph_a:.0f} bar1={bar1:.0f} "
          f"B={ph_b:.0f} bar2={bar2:.0f} | per-iter A={ph_a/len(a):.1f} B={ph_b/len(a):.1f} "
          f"bar={(bar1+bar2)/len(a):.1f}us | nS mean={ns.mean():.0f} max={ns.max():.0f} "
          f"nP mean={a[:, 6].mean():.0f} nC mean={a[:, 7].mean():.0f} nF mean={a[:, 8].mean():.0f} "
          f"fan-phase={fan/len(a):.1f}us/iter", flush=True)
    sm, we, se = a[:, 12], a[:, 13], a[:, 14]
    t0m, ld = a[:, 15], a[:, 16]
    okl = (t0m > 0) & (ld > 0) & (we > 0) & (se > 0)
    if okl.any():
        print(f"   live path (max over warps, from t0): CTA start {np.mean(sm[okl] - t0[okl])/1e3:.2f}us "
              f"item start {np.mean(t0m[okl] - t0[okl])/1e3:.2f}us "
              f"window loaded {np.mean(ld[okl] - t0[okl])/1e3:.2f}us propagated {np.mean(we[okl] - t0[okl])/1e3:.2f}us "
              f"routed {np.mean(se[okl] - t0[okl])/1e3:.2f}us A end {np.mean(ae[okl] - t0[okl])/1e3:.2f}us", flush=True)
    ok = (sm > 0) & (we > 0) & (se > 0)
    if ok.any():
        print(f"   live split per iter: start-skew={np.mean(sm[ok] - t0[ok])/1e3:.2f}us "
              f"work(t0->max work end)={np.mean(we[ok] - t0[ok])/1e3:.2f}us "
              f"scan(->max scan end)={np.mean(se[ok] - we[ok])/1e3:.2f}us "
              f"rest(->A end)={np.mean(ae[ok] - se[ok])/1e3:.2f}us", flush=True)
        t0m, ld = a[:, 15], a[:, 16]
        rt = a[:, 17]
        ok3 = ok & (rt > 0)
        if ok3.any():
            print(f"   routed(before fan-pick completion, max)={np.mean(rt[ok3] - t0[ok3])/1e3:.2f}us "
                  f"scan end(after)={np.mean(se[ok3] - t0[ok3])/1e3:.2f}us", flush=True)
        ok2 = ok & (t0m > 0) & (ld > 0)
        if ok2.any():
            print(f"   setup(t0->max trip0)={np.mean(t0m[ok2] - t0[ok2])/1e3:.2f}us "
                  f"window loaded(max)={np.mean(ld[ok2] - t0[ok2])/1e3:.2f}us "
                  f"propagate(loaded->work end)={np.mean(we[ok2] - ld[ok2])/1e3:.2f}us "
                  f"fan warps end={np.mean(np.where(a[:, 11] > 0, a[:, 11] - t0, 0)[ok2])/1e3:.2f}us", flush=True)


def main():
    from oracle import oracle as O
    from paper_1305_1293_b200 import EngineConfig, run_pch
    from paper_1305_1293_b200 import meshes as M
    name = sys.argv[1]
    specs = sys.argv[2].split(";")
    trace = "--trace" in sys.argv
    m = M.bench_mesh(name)
    if name == "terrain1m":
        src = 354 * 709 + 354
    elif name == "knot4m":
        src = 0
    else:
        src = int(np.argmin(np.linalg.norm(m.positions - m.positions.mean(0), axis=1)))
    t = time.time()
    if "--nocheck" in sys.argv:
        ref = None
        print(f"{name}: F={m.n_faces} src={src} (no oracle check)", flush=True)
    else:
        ref, rs = O.run_ich(m, [src])
        print(f"{name}: F={m.n_faces} src={src} ich={time.time() - t:.2f}s "
              f"ich_windows={rs['total_windows_created']}", flush=True)
        fin = np.isfinite(ref)
    for spec in specs:
        kw = parse(spec)
        env = kw.pop("_env")
        for var in ("PCH_DELTA_MIN", "PCH_DELTA", "PCH_DELTA_MAX"):
            os.environ.pop(var, None)
        os.environ.update(env)
        cfg = EngineConfig(**kw)
        best = None
        for rep in range(3):
            if trace and rep == 2:
                os.environ["PCH_TRACE"] = "/tmp/pch_trace.bin"
            d, st = run_pch(m, [src], cfg)
            os.environ.pop("PCH_TRACE", None)
            if best is None or st.time_kernel_ms < best[1].time_kernel_ms:
                best = (d, st)
        d, st = best
        if ref is None:
            err = float("nan")
        else:
            same = np.array_equal(np.isfinite(d), fin)
            err = float(np.max(np.abs(d[fin] - ref[fin]) / np.maximum(ref[fin], 1e-12))) if same else np.inf
        print(f"{spec:40s} kern={st.time_kernel_ms:8.2f}ms dev={st.time_device_ms:8.2f}ms "
              f"iters={st.iterations:6d} created={st.total_windows_created:10d} "
              f"prop={st.windows_propagated:10d} fans={st.fans_emitted:8d} "
              f"rechk={st.pruned_recheck:8d} regrow={st.buffer_regrows} err={err:.2e}",
              flush=True)
        if trace:
            trace_summary("/tmp/pch_trace.bin")


if __name__ == "__main__":
    main()
