"""Quick GPU-vs-oracle parity and timing sweep (development tool)."""
import sys
import time

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from oracle import oracle as O  # noqa: E402  (checker only)
from paper_1305_1293_b200 import EngineConfig, run_pch  # noqa: E402
from paper_1305_1293_b200 import meshes as M  # noqa: E402
from paper_1305_1293_b200.mesh import build_half_edge_mesh  # noqa: E402


def rel(a, b):
    fa, fb = np.isfinite(a), np.isfinite(b)
    if not np.array_equal(fa, fb):
        return float("inf"), int(np.sum(fa != fb))
    if not fa.any():
        return 0.0, 0
    return float(np.max(np.abs(a[fa] - b[fa]) / np.maximum(np.abs(b[fa]), 1e-12))), 0


def case(name, m, src, ks=(4096,), ich=True):
    t = time.time()
    ref, rs = O.run_ich(m, [src]) if ich else O.run_pch(m, [src], k=4096, workers=8)
    tref = time.time() - t
    for k in ks:
        t = time.time()
        d, st = run_pch(m, [src], EngineConfig(k=k))
        tw = time.time() - t
        t = time.time()
        d, st = run_pch(m, [src], EngineConfig(k=k))
        tw2 = time.time() - t
        e, ninf = rel(d, ref)
        print(f"{name:12s} F={m.n_faces:8d} src={src:7d} k={k:6d} err={e:.2e} infmis={ninf} "
              f"win={st.total_windows_created} (ref {rs['total_windows_created']}) prop={st.windows_propagated} "
              f"iters={st.iterations} fans={st.fans_emitted} rechk={st.pruned_recheck} "
              f"dev={st.time_device_ms:.2f}ms kern={st.time_kernel_ms:.2f}ms wall={tw2*1e3:.1f}ms "
              f"(first {tw*1e3:.0f}ms) ref={tref:.2f}s", flush=True)


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "small"
    if which in ("small", "all"):
        for name, m in M.tiny_corpus().items():
            for s in (0, m.n_vertices // 2):
                case(name, m, s)
        for sub in (2, 3, 4, 5):
            m = build_half_edge_mesh(*M.normalize_edge_scale(*M.icosphere(sub)))
            case(f"ico{sub}", m, 7, ks=(1024, 4096, 65536))
        m = build_half_edge_mesh(*M.terrain(200))
        case("terrain80k", m, 100 * 201 + 100, ks=(1024, 4096, 16384, 65536))
    if which in ("big", "all"):
        m = build_half_edge_mesh(*M.terrain(708))
        case("terrain1m", m, 354 * 709 + 354, ks=(4096, 16384, 65536, 262144))


if __name__ == "__main__":
    main()
