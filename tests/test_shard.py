"""Multi-rank batched rows (paper_1305_1293_b200/shard.py) on CPU: two
gloo ranks, each solving its share of the sources, rows gathered onto
rank 0 in the original order.  The per-rank solve is the CPU oracle here (the GPU
tier runs the same path with run_pch_rows over NCCL)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1305_1293_b200.shard import shard_sources


def test_shard_sources_round_robin():
    parts = [shard_sources(range(10), r, 3).tolist() for r in range(3)]
    assert parts == [[0, 3, 6, 9], [1, 4, 7], [2, 5, 8]]
    assert sorted(sum(parts, [])) == list(range(10))
    assert shard_sources(range(2), 1, 4).tolist() == [1]
    assert shard_sources(range(2), 3, 4).tolist() == []
    with pytest.raises(ValueError):
        shard_sources(range(3), 2, 2)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _oracle_rows(mesh, sources, config):
    from oracle import oracle as O
    return np.stack([O.run_ich(mesh, [int(s)])[0] for s in sources])


def _worker(rank, world, port, sources, out_path):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "tests"))
    import torch.distributed as dist
    from paper_1305_1293_b200 import meshes
    from paper_1305_1293_b200.mesh import build_half_edge_mesh
    from paper_1305_1293_b200.shard import run_rows_sharded
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        m = build_half_edge_mesh(*meshes.normalize_edge_scale(*meshes.icosphere(2)))
        rows = run_rows_sharded(m, sources, solve=_oracle_rows)
        if rows is not None:
            np.save(f"{out_path}.{rank}.npy", rows)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("sources", [[5, 0, 17, 99, 5], [3]])
def test_rows_sharded_gloo_world2(tmp_path, sources):
    from oracle import oracle as O
    from paper_1305_1293_b200 import meshes
    from paper_1305_1293_b200.mesh import build_half_edge_mesh
    out = str(tmp_path / "rows")
    mp.spawn(_worker, args=(2, _free_port(), sources, out), nprocs=2, join=True)
    m = build_half_edge_mesh(*meshes.normalize_edge_scale(*meshes.icosphere(2)))
    ref = np.stack([O.run_ich(m, [s])[0] for s in sources])
    rows = np.load(f"{out}.0.npy")  # gathered onto rank 0 only
    assert rows.shape == (len(sources), m.n_vertices)
    assert np.array_equal(rows, ref)
    assert not os.path.exists(f"{out}.1.npy")
