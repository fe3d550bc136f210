#!/usr/bin/env python
"""Benchmark of the B200 PCH exact-geodesic hot path (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--workload terrain1m|icosphere20k|knot4m|sphere16m|torus500k]

A *step* is one exact single-source geodesic distance field on the
workload mesh (BASELINE.json configs[1]: synthetic noisy heightfield
terrain, 1,002,528 faces, fp64, source at the centre vertex).  The metric
is BASELINE.json's headline: milliseconds per exact single-source field
(lower is better).  With N ranks (torchrun, one process per GPU) every
rank holds a replica of the mesh and computes its own fields -- sources
shard across GPUs with no data-path collective ("scaling": "weak") --
and value = max-over-ranks device time / total fields.

Legs of the b200 arm (one JSON line on rank 0):
  value     device time of the solve with the source list and the output
            field resident in HBM (C ABI pch_run_device), CUDA events on
            the launching stream, L2 flushed (256 MiB write) between steps
            outside the events;
  e2e       the reference-facing call ``run_pch(mesh, [s])`` (host source
            list in, host distance field out; C ABI pch_run), wall clock
            per call, host<->device copies inside;
  roofline  the persistent solver kernel's algorithmic bytes (DESIGN.md
            §4) / its CUDA-event duration vs the measured HBM copy peak;
  cpu_baseline  the CPU port of the reference engine (oracle/, test
            infrastructure) on the host cores, one full field, rank 0 only.

``--impl reference`` times the reference's own CPU algorithm (the C port
of pargeo.engine.run_pch in oracle/, all host threads, reference default
k=4096) on the same workload; rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "ms per exact single-source geodesic field (1M faces)"
UNIT = "ms"

# algorithmic bytes: a stored window is written once and
# read once (SoA record: int32 half-edge + 6 fp64 = 52 B, rounded to the
# 56 B the kernel moves with the key); a propagation reads one 80 B
# half-edge record, three fp64 distances and one 16 B angle-split entry.
BYTES_PER_STORED = 2 * 56
BYTES_PER_PROPAGATED = 80 + 3 * 8 + 16


def _workload(name):
    from paper_1305_1293_b200 import meshes
    m = meshes.bench_mesh(name)
    if name == "terrain1m":
        src = 354 * 709 + 354
    else:
        src = int(np.argmin(np.linalg.norm(m.positions - m.positions.mean(0), axis=1)))
    return m, src


def _peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def _traffic(workload, key=""):
    """dram read+write bytes per launch of the solver kernel (key "") or
    its FP64 pipe utilisation (key "_fp64_pipe") from the committed
    ncu --set full summary, if one exists for this workload."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            t = json.load(f)
        return t.get(workload + key)
    except Exception:
        return None


class Clocks:
    """SM clock / throttle-reason sampling during the timed region
    (B200_PROFILING.md clocks line).  NVML polled from a thread every 2 ms
    (the timed region of a 10-step run is ~0.1 s, too short for
    `nvidia-smi -lms`); nvidia-smi once if NVML is unavailable."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    # nvmlClocksEventReason bits
    BITS = (("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40),
            ("sw_thermal_slowdown", 0x20), ("sw_power_cap", 0x4))

    def __init__(self, index):
        self.index = index
        self.lines = []
        self.thread = None

    def _poll(self):
        import pynvml
        h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
        smax = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        while True:
            sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
            r = pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)
            flags = ["Active" if r & bit else "Not Active" for _, bit in self.BITS]
            self.lines.append(", ".join([str(self.index), str(sm), str(smax), "", ""] + flags))
            if self.stop.wait(0.002):
                return

    def __enter__(self):
        import threading
        try:
            import pynvml
            pynvml.nvmlInit()
            self.stop = threading.Event()
            self.thread = threading.Thread(target=self._poll, daemon=True)
            self.thread.start()
        except Exception:
            self.thread = None
        return self

    def __exit__(self, *exc):
        if self.thread is not None:
            self.stop.set()
            self.thread.join(timeout=5)
        if not self.lines:
            try:
                out = subprocess.run(
                    ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                     "--format=csv,noheader,nounits"],
                    capture_output=True, text=True, timeout=20).stdout
                self.lines = [l for l in out.splitlines() if l.strip()]
            except Exception:
                self.lines = []

    def summary(self):
        sm, smax, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for l in getattr(self, "lines", []):
            c = [x.strip() for x in l.split(",")]
            if len(c) < 9:
                continue
            try:
                sm.append(float(c[1]))
                smax = float(c[2])
            except ValueError:
                continue
            for n, v in zip(names, c[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def _dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _cpu_baseline(mesh, src):
    """The reference engine's CPU port (oracle/pch_oracle.c restating
    pargeo.engine.run_pch, engine.py:433) with all host threads, one full
    field; plus the sequential ICH port (engine.py:624) for context."""
    from oracle import oracle as O
    cores = os.cpu_count() or 1
    t = time.perf_counter()
    ref, st = O.run_pch(mesh, [src], k=4096, workers=cores)
    t_pch = (time.perf_counter() - t) * 1e3
    t = time.perf_counter()
    ich, _ = O.run_ich(mesh, [src])
    t_ich = (time.perf_counter() - t) * 1e3
    return ref, ich, {"value": round(t_pch, 3), "unit": UNIT, "cores": cores, "kind": "port",
                      "sample": f"1 full single-source field, C port of reference run_pch "
                                f"(k=4096, workers={cores})",
                      "ich_1thread_ms": round(t_ich, 3),
                      "windows_propagated": st["windows_propagated"]}


def run_reference(args):
    ws, rank, _ = _dist_env()
    if rank != 0:
        return 0
    from oracle import oracle as O
    mesh, src = _workload(args.workload)
    cores = os.cpu_count() or 1
    tiny_mesh, _ = _workload("icosphere20k") if args.workload != "icosphere20k" else (mesh, src)
    for _ in range(args.warmup):  # warm the thread pool / page in; bounded
        O.run_pch(tiny_mesh, [0], k=4096, workers=cores)
    times = []
    budget_s = args.ref_budget_s
    t_all = time.perf_counter()
    for i in range(args.steps):
        t = time.perf_counter()
        O.run_pch(mesh, [src], k=4096, workers=cores)
        times.append((time.perf_counter() - t) * 1e3)
        if time.perf_counter() - t_all > budget_s:
            break
    ms = float(np.mean(times))
    line = {"impl": "reference", "metric": METRIC, "value": round(ms, 3), "unit": UNIT,
            "n_gpus": ws, "steps": len(times), "warmup": args.warmup, "ms_per_step": round(ms, 3),
            "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": args.workload, "faces": int(mesh.n_faces),
                       "vertices": int(mesh.n_vertices), "source": int(src),
                       "engine": "C port of pargeo run_pch (oracle/pch_oracle.c), k=4096",
                       "l2": "n/a (CPU)"},
            "cpu_baseline": {"value": round(ms, 3), "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": f"{len(times)} full single-source fields"},
            "e2e": {"value": round(ms, 3), "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def _rows_leg(args, ws, rank, local, dev):
    """BASELINE configs[4]: distance-matrix rows on the 500k-face torus,
    sources sharded over the ranks (each GPU a mesh replica, batched rows
    through pch_run_rows), rows all-gathered over NCCL at the end; wall
    time of the whole job (max over ranks), inputs and outputs on the host."""
    import torch
    from paper_1305_1293_b200 import EngineConfig, run_pch_rows
    from paper_1305_1293_b200.shard import gather_rows, shard_sources
    mesh, _ = _workload("torus500k")
    total = args.rows_per_rank * ws
    srcs = np.random.default_rng(4096).choice(mesh.n_vertices, total, replace=False)
    mine = srcs[shard_sources(srcs, rank, ws)]
    cfg = EngineConfig(device=local)
    run_pch_rows(mesh, mine[:32], cfg)  # warm-up: upload, workspace of a full 32-row batch
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize(dev)
    t = time.perf_counter()
    rows, st = run_pch_rows(mesh, mine, cfg)
    if ws > 1:
        gather_rows(rows, total, rank, ws, device=dev)
    torch.cuda.synchronize(dev)
    dt = time.perf_counter() - t
    tt = torch.tensor([dt], dtype=torch.float64, device=dev)
    if ws > 1:
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
    dt = float(tt.item())
    return {"workload": "torus500k", "faces": int(mesh.n_faces), "sources": int(total),
            "sources_per_sec": round(total / dt, 2), "seconds": round(dt, 3), "n_gpus": ws,
            "scaling": "weak", "batch_rows": 32,
            "windows_per_source": int(st.total_windows_created // max(len(mine), 1)),
            "timing": "wall clock, host sources in / host rows out, NCCL all-gather included"}


def _fps_leg(args, ws, rank, local, dev, mesh):
    """North star's second batched workload: greedy geodesic farthest-point
    sampling (pch_fps) on the headline mesh.  Sequential by nature (sample
    s+1 depends on samples 0..s), so N GPUs run N independent samplings
    from different first vertices (weak scaling, no collective); wall time
    of the whole job (max over ranks), host samples + min-field out."""
    import torch
    from paper_1305_1293_b200 import EngineConfig, farthest_point_sampling
    cfg = EngineConfig(device=local)
    first = int(np.random.default_rng(1234 + rank).integers(mesh.n_vertices))
    farthest_point_sampling(mesh, 2, first, cfg)  # warm-up
    # three timed repetitions, median (a sampling run is ~0.1 s of many
    # small solves, so single wall-clock runs vary by +-20 %)
    runs = []
    for _ in range(3):
        if ws > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize(dev)
        t = time.perf_counter()
        samples, _, st = farthest_point_sampling(mesh, args.fps_samples, first, cfg)
        torch.cuda.synchronize(dev)
        runs.append(time.perf_counter() - t)
    dt = statistics.median(runs)
    tt = torch.tensor([dt], dtype=torch.float64, device=dev)
    if ws > 1:
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
    dt = float(tt.item())
    total = args.fps_samples * ws
    return {"workload": args.workload, "samples": int(total), "samples_per_sec": round(total / dt, 2),
            "seconds": round(dt, 3), "n_gpus": ws, "scaling": "weak",
            "seconds_runs": [round(r, 4) for r in runs],
            "windows_propagated_per_sample": int(st.windows_propagated // args.fps_samples),
            "timing": "wall clock (median of 3 runs, max over ranks), one seeded solve + "
                      "device argmax per sample, host results"}


def run_b200(args):
    import torch
    ws, rank, local = _dist_env()
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(local)
    from paper_1305_1293_b200 import EngineConfig, run_pch, run_pch_device
    from paper_1305_1293_b200.engine import device_mesh

    mesh, src = _workload(args.workload)
    cfg = EngineConfig(k=args.k, device=local)
    dm = device_mesh(mesh, local)
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)
    d_src = torch.tensor([src], dtype=torch.int64, device=dev)
    d_out = torch.empty(mesh.n_vertices, dtype=torch.float64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2

    def solve():
        return run_pch_device(mesh, d_src.data_ptr(), 1, d_out.data_ptr(), cfg,
                              stream=stream.cuda_stream)

    for _ in range(args.warmup):
        solve()
    torch.cuda.synchronize(dev)
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize(dev)

    # ---- device-timed leg: inputs resident in HBM ----
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    kern_ms = 0.0
    stored = propagated = created = regrows = iters = 0
    with Clocks(local) as clk:
        for i in range(args.steps):
            flush.zero_()
            evs[i][0].record(stream)
            st = solve()
            evs[i][1].record(stream)
            kern_ms += st.time_kernel_ms
            stored += st.windows_stored
            propagated += st.windows_propagated
            created += st.total_windows_created
            regrows += st.buffer_regrows
            iters += st.iterations
        torch.cuda.synchronize(dev)
    dev_ms = sum(a.elapsed_time(b) for a, b in evs)
    kernel_share = kern_ms / max(dev_ms, 1e-9)
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize(dev)
    field = d_out.cpu().numpy()

    # ---- end-to-end leg: the reference-facing call with host buffers ----
    e2e_ms = 0.0
    for i in range(args.steps):
        torch.cuda.synchronize(dev)
        t = time.perf_counter()
        host, _ = run_pch(mesh, [src], cfg)
        e2e_ms += (time.perf_counter() - t) * 1e3
    if ws > 1:
        torch.distributed.barrier()
    # the default solver reads live tables: repeated solves agree to
    # rounding, not bitwise; flags must be identical
    fin = np.isfinite(field)
    assert np.array_equal(np.isfinite(host), fin), "host and device entry points disagree"
    assert np.all(np.abs(host[fin] - field[fin]) <= 1e-9 * np.maximum(np.abs(field[fin]), 1e-12))

    rows_info = None if args.rows_per_rank <= 0 else _rows_leg(args, ws, rank, local, dev)
    fps_info = None if args.fps_samples <= 0 else _fps_leg(args, ws, rank, local, dev, mesh)

    tot = torch.tensor([dev_ms, e2e_ms, kern_ms], dtype=torch.float64, device=dev)
    if ws > 1:
        torch.distributed.all_reduce(tot, op=torch.distributed.ReduceOp.MAX)
    dev_ms, e2e_ms, kern_ms_max = (float(x) for x in tot.tolist())
    fields = args.steps * ws

    if rank == 0:
        peak, peak_src = _peaks()
        k_ms = kern_ms / args.steps
        alg_bytes = (BYTES_PER_STORED * stored + BYTES_PER_PROPAGATED * propagated) / args.steps
        achieved = alg_bytes / (k_ms * 1e-3) / 1e9
        traffic = _traffic(args.workload)
        line = {
            "metric": METRIC, "value": round(dev_ms / fields, 4), "unit": UNIT, "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(dev_ms / args.steps, 4), "higher_is_better": False,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": args.workload, "faces": int(mesh.n_faces),
                       "vertices": int(mesh.n_vertices), "source": int(src), "k": args.k,
                       "parallelism": f"replicas x{ws} (sources sharded, no collective)",
                       "l2": "flushed (256 MiB write) between steps, outside the events"},
            "e2e": {"value": round(e2e_ms / fields, 4), "unit": UNIT,
                    "h2d_bytes_per_step": 8, "d2h_bytes_per_step": 8 * int(mesh.n_vertices),
                    "call": "paper_1305_1293_b200.run_pch(mesh, [s]) -> C ABI pch_run"},
            "gpu_launches": 4 * (args.steps + regrows),
            "roofline": {"bound": "hbm", "achieved": round(achieved, 2), "peak": peak,
                         "unit": "GB/s", "frac": round(achieved / peak, 5),
                         "traffic": traffic, "kernel": "pch_live",
                         "kernel_ms": round(k_ms, 4),
                         "kernel_share": round(kernel_share, 4),
                         "peak_source": peak_src,
                         "algorithmic_bytes_per_launch": int(alg_bytes),
                         # north star: FP64 pipe utilisation of the propagation
                         # (ncu sm__pipe_fp64_cycles_active, same kernel)
                         "fp64_pipe_frac": _traffic(args.workload, "_fp64_pipe")},
            "windows": {"created_per_field": created // args.steps,
                        "propagated_per_field": propagated // args.steps,
                        "stored_per_field": stored // args.steps,
                        "iterations_per_field": iters // args.steps,
                        "windows_per_sec": round(propagated / (kern_ms * 1e-3), 1)},
            "clocks": clk.summary(),
        }
        if rows_info is not None:
            line["rows"] = rows_info
        if fps_info is not None:
            line["fps"] = fps_info
        if ws == 1 and not args.no_cpu_baseline:
            ref, ich, cb = _cpu_baseline(mesh, src)
            fin = np.isfinite(ref)
            ok = np.array_equal(fin, np.isfinite(field)) and np.array_equal(np.isfinite(ich), fin)
            err = float(np.max(np.abs(field[fin] - ich[fin]) / np.maximum(np.abs(ich[fin]), 1e-12)))
            cb["parity_max_rel_err_vs_ich"] = err
            cb["parity_flags_identical"] = bool(ok)
            line["cpu_baseline"] = cb
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()
    return 0


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("b200", "reference"), default="b200")
    ap.add_argument("--workload", default="terrain1m",
                    choices=("terrain1m", "icosphere20k", "knot4m", "sphere16m", "torus500k"))
    ap.add_argument("--k", type=int, default=16384)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-budget-s", type=float, default=150.0)
    ap.add_argument("--rows-per-rank", type=int, default=64,
                    help="configs[4] distance-matrix rows per GPU (0 = skip)")
    ap.add_argument("--fps-samples", type=int, default=32,
                    help="farthest-point samples per GPU on the headline mesh (0 = skip)")
    args = ap.parse_args(argv)
    if args.warmup < 3 and args.impl == "b200":
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
