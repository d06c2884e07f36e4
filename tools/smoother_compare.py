import sys, json, time
import numpy as np, torch
sys.path.insert(0, '.')
from paper_2112_12397_b200 import api
cfg = int(sys.argv[1])
W = api.Workload(cfg, 42); J = W.system(copy=False)
op = api.BlockSystemOperator(J)
b = torch.tensor(np.random.default_rng(42).uniform(-1, 1, J.total_dimension()), device="cuda", dtype=torch.float64)
for name, amg in [("jacobi", api.AmgConfig(strength_threshold=0.0)),
                  ("cheb2", api.AmgConfig(strength_threshold=0.0, smoother="chebyshev", chebyshev_degree=2)),
                  ("cheb3", api.AmgConfig(strength_threshold=0.0, smoother="chebyshev", chebyshev_degree=3)),
                  ("cheb2_r5", api.AmgConfig(strength_threshold=0.0, smoother="chebyshev", chebyshev_degree=2, chebyshev_ratio=5.0))]:
    for var in ("tup", "tpu"):
        pc = api.GpuPreconditioner.from_host(op, api.HostPreconditioner.from_workload(W, api.PrecondConfig(var, amg=amg)))
        api.gmres(op, pc, b, tol=1e-10, max_iter=20, restart=50, scaled=True)
        x, st = api.gmres(op, pc, b, tol=1e-10, max_iter=500, restart=50, scaled=True)
        pr = pc.profile(5)
        print(json.dumps(dict(config=cfg, smoother=name, variant=var, iters=st.iterations, converged=st.converged,
                              final=st.relative_residuals[-1], solve_s=round(st.device_seconds, 4),
                              apply_ms=round(pr["apply_ms"], 3))), flush=True)
        del pc
