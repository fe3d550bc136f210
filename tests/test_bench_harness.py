"""bench.py's multi-GPU plumbing on CPU: ``--gpus 2`` outside torchrun
re-launches itself under torch.distributed.run (the driver's N>1 path),
the sources shard over the ranks and the rows gather onto rank 0 in source
order (gloo here, NCCL on the GPUs).  ``--dry-run`` replaces the solve by a
placeholder, so no GPU is needed and no number is a measurement."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT


def _run(*extra):
    env = dict(os.environ, MASTER_ADDR="127.0.0.1")
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--dry-run", *extra],
                         capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout  # one JSON line, from rank 0 only
    return json.loads(lines[0])


@pytest.mark.parametrize("gpus,sources", [(1, 7), (2, 10), (2, 7)])
def test_dry_run_shards_and_gathers(gpus, sources):
    line = _run("--gpus", str(gpus), "--rows-sources", str(sources))
    assert line["dry_run"] is True and line["value"] is None
    assert line["n_gpus"] == gpus
    assert line["rows"]["gathered_in_order"] is True
    per = line["rows"]["per_rank"]
    assert sum(per) == sources and max(per) - min(per) <= 1
