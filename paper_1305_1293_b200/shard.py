"""Multi-GPU batched fields: sources shard across ranks, mesh replicated.

A single-source field runs on one GPU.  Batched workloads (distance-matrix
rows, farthest-point sampling rounds) split their sources over the ranks
of one node -- one process per GPU, each holding a replica of the mesh
(``device_mesh``) -- and the rows are gathered once at the end (NCCL over
NVLink on the GPUs, gloo on CPU in the tests).  There is no data-path
collective: ranks never exchange windows or partial fields.

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


def gather_rows(local_rows: np.ndarray, n_total: int, rank: int, world: int,
                device=None) -> np.ndarray | None:
    """Collect every rank's rows (``shard_sources`` order) into the
    original source order on all ranks.  ``local_rows`` is
    ``[len(shard), n_vertices]`` float64."""
    import torch
    import torch.distributed as dist

    nv = local_rows.shape[1] if local_rows.ndim == 2 else 0
    counts = [len(shard_sources(range(n_total), r, world)) for r in range(world)]
    cmax = max(counts) if counts else 0
    dev = device if device is not None else torch.device("cpu")
    buf = torch.full((cmax, nv), float("nan"), dtype=torch.float64, device=dev)
    if len(local_rows):
        buf[: len(local_rows)] = torch.as_tensor(local_rows, dtype=torch.float64, device=dev)
    outs = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(outs, buf)
    rows = np.empty((n_total, nv), dtype=np.float64)
    for r in range(world):
        idx = shard_sources(range(n_total), r, world)
        rows[idx] = outs[r][: counts[r]].cpu().numpy()
    return rows


def run_rows_sharded(mesh, sources, config=None, solve=None, device=None):
    """Distance-matrix rows for ``sources`` computed by all ranks of the
    initialised process group; every rank returns the full
    ``[len(sources), n_vertices]`` array.  ``solve(mesh, sources, config)``
    defaults to the GPU ``run_pch_rows`` on this rank's device."""
    import torch.distributed as dist

    world = dist.get_world_size() if dist.is_initialized() else 1
    rank = dist.get_rank() if dist.is_initialized() else 0
    src = np.asarray([int(s) for s in sources], dtype=np.int64)
    mine = src[shard_sources(src, rank, world)]
    if solve is None:
        from .engine import run_pch_rows
        solve = lambda m, s, c: run_pch_rows(m, s, c)[0]  # noqa: E731
    local = solve(mesh, mine, config) if len(mine) else np.empty((0, mesh.n_vertices))
    if world == 1:
        return np.asarray(local)
    return gather_rows(np.asarray(local), len(src), rank, world, device)
