"""A short GMRES solve on a BASELINE config (for ncu launch lists of the whole iteration; run ncu with
--profile-from-start off: only the second solve is inside cudaProfilerStart / Stop).

    python tools/profile_solve.py [config] [variant] [max_iter] [mgs|cgs] [ordered|strided]
"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_2112_12397_b200 import api  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
var = sys.argv[2] if len(sys.argv) > 2 else "tup"
its = int(sys.argv[3]) if len(sys.argv) > 3 else 10
orth = sys.argv[4] if len(sys.argv) > 4 else "cgs"
row_sum = sys.argv[5] if len(sys.argv) > 5 else "strided"
W = api.Workload(cfg, 42)
J = W.system(copy=False)  # views (config 5: no 30 GB copy); the preconditioner is built on the workload in place
op = api.BlockSystemOperator(J)
pc = api.GpuPreconditioner.from_host(op, api.HostPreconditioner.from_workload(W, api.PrecondConfig(
    var, amg=api.AmgConfig(strength_threshold=0.0, row_sum=row_sum))))
b = torch.tensor(np.random.default_rng(42).uniform(-1, 1, J.total_dimension()), device="cuda", dtype=torch.float64)
x, st = api.gmres(op, pc, b, tol=1e-10, max_iter=its, restart=50, scaled=True, orthogonalization=orth)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()  # ncu --profile-from-start off captures only this solve
t0 = time.perf_counter()
x, st = api.gmres(op, pc, b, tol=1e-10, max_iter=its, restart=50, scaled=True, orthogonalization=orth)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
wall = time.perf_counter() - t0
print(f"iters {st.iterations} device {st.device_seconds * 1e3:.2f} ms wall {wall * 1e3:.2f} ms "
      f"per-iter {st.device_seconds / max(1, st.iterations) * 1e3:.3f} ms launches {st.kernel_launches}")
