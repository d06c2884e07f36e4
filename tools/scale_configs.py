"""Measure larger BASELINE configs: generation / setup time, hierarchy, apply and solve timings.

    python tools/scale_configs.py 3 [4 ...]
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_2112_12397_b200 import api  # noqa: E402

hbm = 6548.8
for cfg in [int(a) for a in sys.argv[1:]]:
    t0 = time.perf_counter()
    W = api.Workload(cfg, 42)
    J = W.system()
    gen = time.perf_counter() - t0
    t0 = time.perf_counter()
    op = api.BlockSystemOperator(J)
    hp = api.HostPreconditioner(J, api.PrecondConfig("tup", amg=api.AmgConfig(strength_threshold=0.0),
                                                  factor_solve=os.environ.get("FS", "auto")))
    host_setup = time.perf_counter() - t0
    t0 = time.perf_counter()
    pc = api.GpuPreconditioner.from_host(op, hp)
    upload = time.perf_counter() - t0
    del hp
    pr = pc.profile(10)
    b = torch.tensor(np.random.default_rng(42).uniform(-1, 1, J.total_dimension()), device="cuda", dtype=torch.float64)
    x, st = api.gmres(op, pc, b, tol=1e-10, max_iter=100, restart=50, scaled=True)
    free, total = torch.cuda.mem_get_info()
    print(json.dumps(dict(config=cfg, factor_solve=pc.factor_solve, n_u=J.n_u, n_t=J.n_t, n_p=J.n_p, info=W.info(), generate_s=round(gen, 1),
                          host_setup_s=round(host_setup, 1), upload_s=round(upload, 1), levels=pr["level_rows"],
                          level_nnz=pr["level_nnz"], apply_ms=round(pr["apply_ms"], 3),
                          apply_GBps=round(pr["apply_bytes"] / pr["apply_ms"] / 1e6, 1),
                          apply_frac=round(pr["apply_bytes"] / pr["apply_ms"] / 1e6 / hbm, 3),
                          fine_post_GBps=round(pr["fine_post_bytes"] / pr["fine_post_ms"] / 1e6, 1),
                          fine_resid_GBps=round(pr["fine_resid_bytes"] / pr["fine_resid_ms"] / 1e6, 1),
                          japply_GBps=round(pr["japply_bytes"] / pr["japply_ms"] / 1e6, 1),
                          band_ms=round(pr["band_ms"], 3), iters100_s=round(st.device_seconds, 3),
                          per_iter_ms=round(st.device_seconds / max(1, st.iterations) * 1e3, 3),
                          final_100=st.relative_residuals[-1], gpu_mem_used_GB=round((total - free) / 1e9, 1))),
          flush=True)
    del pc, op, J, W
    torch.cuda.empty_cache()
