#!/usr/bin/env python
"""Benchmark of the B200 PCH exact-geodesic hot path (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--workload terrain1m|icosphere20k|knot4m|sphere16m|torus500k]
                    [--rows-sources 4096] [--fps-samples 32] [--dry-run]

A *step* is one exact single-source geodesic distance field on the
workload mesh (BASELINE.json configs[1]: synthetic noisy heightfield
terrain, 1,002,528 faces, fp64).  The metric is BASELINE.json's headline:
milliseconds per exact single-source field (lower is better).

Multi-GPU: ``--gpus N`` without a torchrun environment re-launches itself
under ``torch.distributed.run`` with N ranks (one process per GPU, NCCL).
Every rank holds a replica of the mesh.  Single-source fields: rank r
solves its own source (the r-th nearest vertex to the centre, so every
rank's field costs about the same; "scaling": "weak") and ``value`` is the
per-field device time, max over ranks -- a per-GPU latency, not divided
by N.  Distance-matrix rows (configs[4]): 4096 sources on the 500k-face
torus sharded over the ranks (strong scaling), each rank's rows written
to its HBM by pch_run_rows_device and gathered onto rank 0 over NCCL
device to device; sources/s = 4096 / max-over-ranks time.

Legs of the b200 arm (one JSON line on rank 0):
  value     device time of the solve with the source list and the output
            field resident in HBM (C ABI pch_run_device), CUDA events on
            the launching stream, L2 flushed (256 MiB write) between steps
            outside the events;
  e2e       the reference-facing call ``run_pch(mesh, [s])`` (host source
            list in, host distance field out; C ABI pch_run), wall clock
            per call, host<->device copies inside;
  roofline  the solver kernel (pch_live): algorithmic bytes
            per launch / its CUDA-event time against the measured HBM copy
            peak; measured DRAM bytes (committed ncu capture, rejected when
            the kernel sources changed since); the latency roofline
            (iterations x (grid barrier + mean batch work item), both
            measured in this run) -- the bound that applies; FP64 peak
            measured in this run (pch_probe);
  rows      configs[4] throughput with its own roofline;
  fps       farthest-point samples/s;
  cpu_baseline  the CPU port of the reference engine (oracle/, test
            infrastructure) on the host cores, one full field, rank 0 only.

``--impl reference`` times the reference's own CPU algorithm (the C port
of pargeo.engine.run_pch in oracle/, all host threads, reference default
k=4096) on the same workload; rank 0 only.  ``--dry-run`` drives the
launcher, sharding and gather plumbing on CPU (gloo) without a GPU and
prints a line marked ``"dry_run": true`` (tests/test_bench_harness.py).
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import socket
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
ROWS_SOURCES = 4096  # BASELINE configs[4]

# algorithmic bytes: a stored window is written once and
# read once (SoA record: int4 half-edges/vertices 16 B + uint2 apex/row 8 B
# + six fp64 48 B = 72 B); a propagation reads one 64 B FaceRec, three
# fp64 distances and one 16 B angle-split entry.
BYTES_PER_STORED = 2 * 72
BYTES_PER_PROPAGATED = 64 + 3 * 8 + 16
KERNEL_SOURCES = ("paper_1305_1293_b200/csrc/pch_engine.cu", "paper_1305_1293_b200/csrc/pch_device.cuh")


def kernel_sha() -> str:
    """Digest of the solver's sources: a committed ncu capture applies only
    to the build it was taken on."""
    h = hashlib.sha256()
    for rel in KERNEL_SOURCES:
        with open(os.path.join(ROOT, rel), "rb") as f:
            h.update(f.read())
    return h.hexdigest()[:16]


def _workload(name):
    from paper_1305_1293_b200 import meshes
    m = meshes.bench_mesh(name)
    if name == "terrain1m":
        src = 354 * 709 + 354
    else:
        src = int(np.argmin(np.linalg.norm(m.positions - m.positions.mean(0), axis=1)))
    return m, src


def _rank_source(mesh, centre, rank):
    """Rank r's source: the r-th nearest vertex to the centre source
    (distinct per rank, about the same field cost)."""
    if rank == 0:
        return int(centre)
    d = np.linalg.norm(mesh.positions - mesh.positions[centre], axis=1)
    return int(np.argsort(d, kind="stable")[rank])


def _peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def _ncu(key):
    """An entry of the committed ncu --set full summary
    (profiles/ncu_traffic.json): (value, status).  Entries carry the
    kernel_sha() of the build they were captured on; a stale one is not
    reported."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            t = json.load(f)
    except Exception:
        return None, "no capture"
    e = t.get(key)
    if not isinstance(e, dict):
        return None, "no capture"
    if e.get("kernel_sha") != kernel_sha():
        return None, f"stale (captured on {e.get('kernel_sha')}, build {kernel_sha()})"
    return e, "current"


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


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _launch(args, argv):
    """--gpus N outside torchrun: re-launch this script with N ranks."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={_free_port()}", os.path.abspath(__file__), *argv]
    return subprocess.call(cmd)


def _max_over_ranks(vals, ws, dev):
    import torch
    t = torch.tensor(vals, dtype=torch.float64, device=dev)
    if ws > 1:
        import torch.distributed as dist
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(x) for x in t.tolist()]


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
    """BASELINE configs[4]: 4096 distance-matrix rows on the 500k-face
    torus, sources sharded over the ranks (each GPU a mesh replica), this
    rank's rows written to its HBM by pch_run_rows_device, gathered onto
    rank 0 over NCCL device to device, then one copy to the host on rank 0.
    Device time (CUDA events, solve + gather) max over ranks; the host copy
    is reported beside it."""
    import torch
    from paper_1305_1293_b200 import EngineConfig, run_pch, run_pch_rows_device
    from paper_1305_1293_b200.shard import gather_rows, shard_sources
    mesh, _ = _workload("torus500k")
    total = args.rows_sources
    srcs = np.random.default_rng(4096).choice(mesh.n_vertices, total, replace=False)
    mine = srcs[shard_sources(srcs, rank, ws)]
    cfg = EngineConfig(device=local)
    stream = torch.cuda.current_stream(dev)
    d_src = torch.as_tensor(mine, device=dev)
    out = torch.empty((len(mine), mesh.n_vertices), dtype=torch.float64, device=dev)
    # warm-up: mesh upload and the workspace of a full 32-row batch
    run_pch_rows_device(mesh, d_src.data_ptr(), min(32, len(mine)), out.data_ptr(), cfg,
                        stream=stream.cuda_stream)
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize(dev)
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    with Clocks(local) as clk:
        e0.record(stream)
        st = run_pch_rows_device(mesh, d_src.data_ptr(), len(mine), out.data_ptr(), cfg,
                                 stream=stream.cuda_stream)
        e1.record(stream)
        full = gather_rows(out, total, rank, ws) if ws > 1 else out
        e2.record(stream)
        torch.cuda.synchronize(dev)
    solve_s, gather_s = e0.elapsed_time(e1) / 1e3, e1.elapsed_time(e2) / 1e3
    host_s = 0.0
    check = None
    if rank == 0:
        t = time.perf_counter()
        host = full.cpu().numpy()
        host_s = time.perf_counter() - t
        # parity of the batched path: rows 1 and 2 (oracle rounding holes
        # there) against single-source fields of the same sources
        errs = []
        for r in (1, 2):
            one, _ = run_pch(mesh, [int(srcs[r])], cfg)
            fin = np.isfinite(one)
            same = np.array_equal(fin, np.isfinite(host[r]))
            errs.append(float(np.max(np.abs(host[r][fin] - one[fin]) / np.maximum(one[fin], 1e-12)))
                        if same else float("inf"))
        check = max(errs)
        del host
    tot_s, solve_s, gather_s, kern_ms = _max_over_ranks(
        [solve_s + gather_s, solve_s, gather_s, st.time_kernel_ms], ws, dev)
    peak, _ = _peaks()
    alg = BYTES_PER_STORED * st.windows_stored + BYTES_PER_PROPAGATED * st.windows_propagated
    achieved = alg / (st.time_kernel_ms * 1e-3) / 1e9
    ncu, ncu_status = _ncu("rows_torus500k")
    info = {"workload": "torus500k", "faces": int(mesh.n_faces), "sources": int(total),
            "sources_per_sec": round(total / tot_s, 2), "seconds": round(tot_s, 3),
            "solve_seconds": round(solve_s, 3), "gather_seconds": round(gather_s, 3),
            "host_copy_seconds": round(host_s, 3), "n_gpus": ws, "scaling": "strong",
            "batch_rows": 32, "windows_per_source": int(st.total_windows_created // max(len(mine), 1)),
            "parity_rows_vs_single_max_rel_err": check,
            "roofline": {"bound": "latency", "achieved": round(achieved, 2), "peak": peak,
                         "unit": "GB/s", "frac": round(achieved / peak, 5),
                         "traffic": ncu.get("dram_bytes") if ncu else None,
                         "traffic_status": ncu_status, "kernel": "pch_live (batched rows)",
                         "kernel_ms_rank0": round(st.time_kernel_ms, 2)},
            "clocks": clk.summary(),
            "timing": "CUDA events on the launching stream: rows solve (sources resident) + "
                      "NCCL gather onto rank 0, max over ranks; host copy of the full matrix on "
                      "rank 0 reported separately"}
    if ncu:
        info["roofline"]["dram_frac"] = round(ncu["dram_bytes"] / (ncu["kernel_ms"] * 1e-3) / 1e9 / peak, 5)
    return info


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


def run_dry(args):
    """Launcher / sharding / gather plumbing without a GPU (gloo): each
    rank fills its rows with a placeholder (Euclidean distance from the
    source -- not a solve), rank 0 checks the gathered order and prints a
    line marked dry_run.  Covered by tests/test_bench_harness.py."""
    import torch
    import torch.distributed as dist
    from paper_1305_1293_b200 import meshes
    from paper_1305_1293_b200.mesh import build_half_edge_mesh
    from paper_1305_1293_b200.shard import gather_rows, shard_sources
    ws, rank, _ = _dist_env()
    if ws > 1:
        dist.init_process_group("gloo")
    m = build_half_edge_mesh(*meshes.normalize_edge_scale(*meshes.icosphere(2)))
    total = args.rows_sources
    srcs = np.random.default_rng(4096).choice(m.n_vertices, total, replace=total > m.n_vertices)
    mine = srcs[shard_sources(srcs, rank, ws)]
    local = torch.as_tensor(np.stack([np.linalg.norm(m.positions - m.positions[s], axis=1) for s in mine])
                            if len(mine) else np.empty((0, m.n_vertices)))
    full = gather_rows(local, total, rank, ws) if ws > 1 else local
    if rank == 0:
        want = np.stack([np.linalg.norm(m.positions - m.positions[s], axis=1) for s in srcs])
        ok = bool(np.array_equal(full.numpy(), want))
        print(json.dumps({"dry_run": True, "metric": METRIC, "value": None, "unit": UNIT,
                          "n_gpus": ws, "rows": {"sources": int(total), "gathered_in_order": ok,
                                                 "per_rank": [len(shard_sources(srcs, r, ws))
                                                              for r in range(ws)]}}), flush=True)
    if ws > 1:
        dist.destroy_process_group()
    return 0


def run_b200(args):
    import torch
    ws, rank, local = _dist_env()
    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_1305_1293_b200 import EngineConfig, run_pch, run_pch_device
    from paper_1305_1293_b200.engine import device_mesh, probe

    mesh, centre = _workload(args.workload)
    src = _rank_source(mesh, centre, rank)
    cfg = EngineConfig(k=args.k, device=local)
    device_mesh(mesh, local)
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
    stored = propagated = created = regrows = iters = barriers = 0
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
            barriers += st.grid_barriers
        torch.cuda.synchronize(dev)
    dev_ms = sum(a.elapsed_time(b) for a, b in evs)
    kernel_share = kern_ms / max(dev_ms, 1e-9)
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize(dev)
    field = d_out.cpu().numpy()

    # ---- end-to-end leg: the reference-facing call with host buffers ----
    e2e_ms = 0.0
    host = None
    for i in range(args.warmup + args.steps):  # warm-up calls untimed, like the device leg
        torch.cuda.synchronize(dev)
        t = time.perf_counter()
        host, _ = run_pch(mesh, [src], cfg)
        if i >= args.warmup:
            e2e_ms += (time.perf_counter() - t) * 1e3
    if ws > 1:
        torch.distributed.barrier()
    # the default solver reads live tables: repeated solves agree to
    # rounding, not bitwise; flags must be identical
    fin = np.isfinite(field)
    assert np.array_equal(np.isfinite(host), fin), "host and device entry points disagree"
    assert np.all(np.abs(host[fin] - field[fin]) <= 1e-9 * np.maximum(np.abs(field[fin]), 1e-12))

    # one more solve with the phase attribution on (untimed: it costs ~3 %):
    # the RunStats phase split and the mean batch work item of the latency
    # roofline
    from dataclasses import replace
    stp = run_pch_device(mesh, d_src.data_ptr(), 1, d_out.data_ptr(), replace(cfg, phase_times=True),
                         stream=stream.cuda_stream)
    phase = [stp.time_select, stp.time_propagate, stp.time_compact, stp.time_events]
    item_us = stp.prop_item_us
    pr = probe(local)
    rows_info = None if args.rows_sources <= 0 else _rows_leg(args, ws, rank, local, dev)
    fps_info = None if args.fps_samples <= 0 else _fps_leg(args, ws, rank, local, dev, mesh)

    dev_ms, e2e_ms, kern_ms_max = _max_over_ranks([dev_ms, e2e_ms, kern_ms], ws, dev)

    if rank == 0:
        peak, peak_src = _peaks()
        k_ms = kern_ms / args.steps
        it = iters / args.steps
        alg_bytes = (BYTES_PER_STORED * stored + BYTES_PER_PROPAGATED * propagated) / args.steps
        achieved = alg_bytes / (k_ms * 1e-3) / 1e9
        ncu, ncu_status = _ncu(args.workload)
        us_iter = k_ms * 1e3 / max(it, 1)
        bar_per_it = barriers / max(iters, 1)
        floor_iter = bar_per_it * pr["grid_barrier_us"] + item_us
        roof = {"bound": "latency", "achieved": round(achieved, 2), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 5),
                "traffic": ncu.get("dram_bytes") if ncu else None, "traffic_status": ncu_status,
                "kernel": "pch_live", "kernel_ms": round(k_ms, 4),
                "kernel_share": round(kernel_share, 4), "peak_source": peak_src,
                "algorithmic_bytes_per_launch": int(alg_bytes),
                "bytes_per_unit": {"stored_window": BYTES_PER_STORED,
                                   "propagation": BYTES_PER_PROPAGATED},
                # the bound that applies: iterations x (grid barrier + one
                # batch work item), both measured in this run
                "latency": {"iterations": round(it, 1), "us_per_iteration": round(us_iter, 3),
                            "grid_barrier_us": round(pr["grid_barrier_us"], 3),
                            "grid_barriers_per_iteration": round(bar_per_it, 3),
                            "mean_item_us": round(item_us, 3),
                            "floor_us_per_iteration": round(floor_iter, 3),
                            "frac": round(floor_iter / us_iter, 4)},
                "fp64": {"peak_tflops_measured": round(pr["fp64_tflops"], 2),
                         "pipe_frac_ncu": ncu.get("fp64_pipe_frac") if ncu else None},
                "phase_ms": dict(zip(("select", "propagate", "compact", "events"),
                                     (round(x * 1e3, 4) for x in phase)))}
        if ncu:
            roof["dram_frac"] = round(ncu["dram_bytes"] / (k_ms * 1e-3) / 1e9 / peak, 5)
        line = {
            "metric": METRIC, "value": round(dev_ms / args.steps, 4), "unit": UNIT, "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(dev_ms / args.steps, 4), "higher_is_better": False,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": args.workload, "faces": int(mesh.n_faces),
                       "vertices": int(mesh.n_vertices), "source": int(centre), "k": args.k,
                       "parallelism": f"replicas x{ws} (one source per rank, no collective)",
                       "l2": "flushed (256 MiB write) between steps, outside the events"},
            "e2e": {"value": round(e2e_ms / args.steps, 4), "unit": UNIT,
                    "h2d_bytes_per_step": 8, "d2h_bytes_per_step": 8 * int(mesh.n_vertices),
                    "call": "paper_1305_1293_b200.run_pch(mesh, [s]) -> C ABI pch_run"},
            "gpu_launches": 4 * (args.steps + regrows),
            "roofline": roof,
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
    argv = list(sys.argv[1:] if argv is None else argv)
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("b200", "reference"), default="b200")
    ap.add_argument("--workload", default="terrain1m",
                    choices=("terrain1m", "icosphere20k", "knot4m", "knotg4m", "sphere16m", "torus500k"))
    ap.add_argument("--k", type=int, default=16384)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-budget-s", type=float, default=150.0)
    ap.add_argument("--rows-sources", type=int, default=ROWS_SOURCES,
                    help="configs[4] distance-matrix rows in total, sharded over the GPUs (0 = skip)")
    ap.add_argument("--fps-samples", type=int, default=32,
                    help="farthest-point samples per GPU on the headline mesh (0 = skip)")
    ap.add_argument("--dry-run", action="store_true",
                    help="launcher/shard/gather plumbing on CPU (gloo), no GPU, no measurement")
    args = ap.parse_args(argv)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return _launch(args, argv)
    if args.warmup < 3 and args.impl == "b200":
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    if args.dry_run:
        return run_dry(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
