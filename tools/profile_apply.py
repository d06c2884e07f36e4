"""One preconditioner apply (+ one J apply) on a BASELINE config, for ncu launch lists.

    python tools/profile_apply.py [config] [variant] [reps] [ordered|strided]
Warm-up applies run first; profile the last `reps` with ncu -s <skip>.
"""
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_2112_12397_b200 import api  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
var = sys.argv[2] if len(sys.argv) > 2 else "tup"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
row_sum = sys.argv[4] if len(sys.argv) > 4 else "ordered"
J = api.Workload(cfg, 42).system()
op = api.BlockSystemOperator(J)
pc = api.GpuPreconditioner.from_host(op, api.HostPreconditioner(J, api.PrecondConfig(
    var, amg=api.AmgConfig(strength_threshold=0.0, row_sum=row_sum))))
x = torch.tensor(np.random.default_rng(0).uniform(-1, 1, J.total_dimension()), device="cuda", dtype=torch.float64)
for _ in range(2 + reps):
    y = pc.apply(x)
    z = op.apply(x)
torch.cuda.synchronize()
print("levels", pc.profile(3)["level_rows"], "launches per apply", pc.traffic()["apply_launches"])
