"""Multi-GPU batched fields: sources shard across ranks, mesh replicated.

A single-source field runs on one GPU.  Batched workloads (distance-matrix
rows, farthest-point sampling rounds) split their sources over the ranks
of one node -- one process per GPU, each holding a replica of the mesh
(``device_mesh``) -- and the rows are gathered once at the end onto rank 0
(NCCL over NVLink on the GPUs, device memory to device memory; gloo on CPU
in the tests).  There is no data-path collective: ranks never exchange
windows or partial fields.

Reference context: the reference computes multi-source fields and
repeated single-source runs on one host (engine.py:433, cli.py:103,
paper Table 3); the sharding is the B200 design's scale-out.
"""
from __future__ import annotations

import numpy as np


def shard_sources(sources, rank: int, world: int) -> np.ndarray:
    """Indices (into ``sources``) owned by ``rank``: round-robin, so every
    rank gets the same count +-1 and similar source distributions."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank/world {rank}/{world}")
    n = len(sources)
    return np.arange(rank, n, world, dtype=np.int64)


def gather_rows(local, n_total: int, rank: int, world: int):
    """Collect every rank's rows (``shard_sources`` order) onto rank 0 in
    the original source order.  ``local`` is a ``[len(shard), n_vertices]``
    float64 torch tensor on this rank's device (NCCL) or on the CPU (gloo);
    rank 0 returns the ``[n_total, n_vertices]`` tensor on the same device,
    the other ranks ``None``.  One point-to-point transfer per rank into
    rank 0, no host round trip."""
    import torch
    import torch.distributed as dist

    nv = int(local.shape[1])
    counts = [len(shard_sources(range(n_total), r, world)) for r in range(world)]
    cmax = max(counts)
    if local.shape[0] < cmax:  # equal-size buffers for the collective
        pad = torch.full((cmax - local.shape[0], nv), float("nan"), dtype=local.dtype,
                         device=local.device)
        local = torch.cat([local, pad])
    # point-to-point into rank 0 (NCCL send/recv over NVLink; gloo on CPU),
    # all transfers posted at once
    local = local.contiguous()
    if rank != 0:
        for w in dist.batch_isend_irecv([dist.P2POp(dist.isend, local, 0)]):
            w.wait()
        return None
    bufs = [local] + [torch.empty_like(local) for _ in range(1, world)]
    ops = [dist.P2POp(dist.irecv, bufs[r], r) for r in range(1, world)]
    for w in dist.batch_isend_irecv(ops):
        w.wait()
    out = torch.empty((n_total, nv), dtype=local.dtype, device=local.device)
    for r in range(world):
        idx = torch.as_tensor(shard_sources(range(n_total), r, world), device=local.device)
        if len(idx):
            out.index_copy_(0, idx, bufs[r][: counts[r]])
    return out


def run_rows_sharded(mesh, sources, config=None, solve=None):
    """Distance-matrix rows for ``sources`` computed by all ranks of the
    initialised process group (or this process alone); rank 0 returns the
    full ``[len(sources), n_vertices]`` float64 numpy array, the other
    ranks ``None``.  The default ``solve`` is the GPU path: this rank's
    share through ``run_pch_rows_device`` into device memory, gathered over
    NCCL device to device; ``solve(mesh, sources, config) -> array`` (the
    CPU tests' oracle) is gathered over gloo."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size() if dist.is_initialized() else 1
    rank = dist.get_rank() if dist.is_initialized() else 0
    src = np.asarray([int(s) for s in sources], dtype=np.int64)
    mine = src[shard_sources(src, rank, world)]
    if solve is None:
        from .engine import EngineConfig, run_pch_rows_device
        config = config or EngineConfig()
        dev = torch.device("cuda", config.device)
        local = torch.empty((len(mine), mesh.n_vertices), dtype=torch.float64, device=dev)
        if len(mine):
            d_src = torch.as_tensor(mine, device=dev)
            run_pch_rows_device(mesh, d_src.data_ptr(), len(mine), local.data_ptr(), config,
                                stream=torch.cuda.current_stream(dev).cuda_stream)
    else:
        rows = solve(mesh, mine, config) if len(mine) else np.empty((0, mesh.n_vertices))
        local = torch.as_tensor(np.asarray(rows, dtype=np.float64))
    if world == 1:
        return local.cpu().numpy()
    out = gather_rows(local, len(src), rank, world)
    return None if out is None else out.cpu().numpy()
