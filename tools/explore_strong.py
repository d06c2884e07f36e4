"""Exploration: strong inner AMG settings (reference AmgConfig knobs) on BASELINE config 2."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_2112_12397_b200 import api  # noqa: E402

J = api.Workload(2, 42).system()
op = api.BlockSystemOperator(J)
b = torch.tensor(np.random.default_rng(42).uniform(-1, 1, J.total_dimension()), device="cuda", dtype=torch.float64)
for var, pre, cyc, restart in (("tup", 3, 2, 50), ("tup", 3, 3, 50), ("tup", 5, 2, 50), ("tup", 2, 4, 50),
                               ("tpu", 3, 2, 50), ("tup", 1, 1, 500), ("tup", 3, 2, 500)):
    hp = api.HostPreconditioner(J, api.PrecondConfig(var, amg=api.AmgConfig(strength_threshold=0.0, pre_sweeps=pre,
                                                                           post_sweeps=pre, cycles_per_apply=cyc)))
    pc = api.GpuPreconditioner.from_host(op, hp)
    x, st = api.gmres(op, pc, b, tol=1e-10, max_iter=500, restart=restart, scaled=True)
    pr = pc.profile(5)
    print(json.dumps(dict(var=var, sweeps=pre, cycles=cyc, restart=restart, iters=st.iterations, conv=st.converged,
                          final=st.relative_residuals[-1], solve_s=round(st.device_seconds, 3),
                          apply_ms=round(pr["apply_ms"], 3))), flush=True)
    del pc, hp
