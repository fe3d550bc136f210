import sys, numpy as np
sys.path.insert(0, '/root/repo')
from paper_1305_1293_b200 import EngineConfig, run_pch
from paper_1305_1293_b200 import meshes as M
m = M.bench_mesh("knot4m")
d, st = run_pch(m, [0], EngineConfig(k=65536))
np.save('/root/repo/gpurun_out/knot4m_gpu.npy', d)
print(st.time_kernel_ms, st.iterations, int(np.sum(~np.isfinite(d))))
