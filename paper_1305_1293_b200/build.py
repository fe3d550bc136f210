"""In-tree build of the CUDA library (sm_100a) -- no JIT cache, so the
``.so`` travels with the repository snapshot to the GPU box."""
from __future__ import annotations

import os
import shutil
import subprocess

_HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(_HERE)
CSRC = os.path.join(_HERE, "csrc")
OUT = os.path.join(_HERE, "_lib", "libpch_b200.so")

SOURCES = ["pch_engine.cu", "pch_mesh.cpp"]
DEPS = ["pch_device.cuh", os.path.join(ROOT, "include", "pch_b200.h")]

NVCC_FLAGS = ["-std=c++17", "-O3", "-lineinfo",
              "-gencode", "arch=compute_100a,code=sm_100a",
              "-Xcompiler", "-fPIC,-ffp-contract=off", "-shared", "-Xptxas", "-v"]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    paths = [os.path.join(CSRC, s) for s in SOURCES]
    paths += [d if os.path.isabs(d) else os.path.join(CSRC, d) for d in DEPS]
    return any(os.path.getmtime(p) > t for p in paths)


def build_native(force: bool = False, verbose: bool = False) -> str:
    """Compile csrc/*.cu into _lib/libpch_b200.so for sm_100a."""
    if not force and not _stale():
        return OUT
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    cmd = [_nvcc(), *NVCC_FLAGS, "-o", OUT + ".tmp",
           *[os.path.join(CSRC, s) for s in SOURCES]]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + res.stdout + res.stderr)
    os.replace(OUT + ".tmp", OUT)
    if verbose:
        print(res.stderr)
    return OUT


if __name__ == "__main__":
    print(build_native(force=True, verbose=True))
