"""Large BASELINE configs (4, 5) through the lean host path: the generated system is viewed, not copied, and the
preconditioner is built on the workload in place (fp_workload_host_precond_build).  Prints one JSON line with
setup phases, host peak RSS, the apply profile and a short GMRES(50) run.

    FRACPREC_B200_VERBOSE=1 python tools/big_config.py 5 [gmres_iters] [ordered|strided]
The GMRES run is timed with classical (cgs) and modified (mgs) Gram-Schmidt.
"""
import json
import os
import resource
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2112_12397_b200 import api  # noqa: E402

cfg = int(sys.argv[1])
its = int(sys.argv[2]) if len(sys.argv) > 2 else 50
row_sum = sys.argv[3] if len(sys.argv) > 3 else "strided"
_peaks = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
hbm = json.load(open(_peaks))["hbm_gbs"] if os.path.exists(_peaks) else 6650.0  # else B200_PROFILING.md fallback


def rss_gb():
    return resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 1e6


out = {"config": cfg}
t0 = time.perf_counter()
W = api.Workload(cfg, 42)
J = W.system(copy=False)
out["generate_s"], out["rss_after_generate_GB"] = round(time.perf_counter() - t0, 1), round(rss_gb(), 1)
print(json.dumps(out), flush=True)
t0 = time.perf_counter()
hp = api.HostPreconditioner.from_workload(W, api.PrecondConfig("tup", amg=api.AmgConfig(strength_threshold=0.0,
                                                                                       row_sum=row_sum)))
out["row_sum"] = row_sum
out["host_setup_s"], out["rss_after_setup_GB"] = round(time.perf_counter() - t0, 1), round(rss_gb(), 1)
out["levels"] = hp.level_sizes()
print(json.dumps(out), flush=True)
t0 = time.perf_counter()
op = api.BlockSystemOperator(J)
out["system_upload_s"] = round(time.perf_counter() - t0, 1)
t0 = time.perf_counter()
pc = api.GpuPreconditioner.from_host(op, hp)
out["precond_upload_s"], out["rss_after_upload_GB"] = round(time.perf_counter() - t0, 1), round(rss_gb(), 1)
del hp
out["factor_solve"] = pc.factor_solve
free, total = torch.cuda.mem_get_info()
out["gpu_mem_used_GB"] = round((total - free) / 1e9, 1)
print(json.dumps(out), flush=True)
pr = pc.profile(5)
out.update(n=J.total_dimension(), apply_ms=round(pr["apply_ms"], 3),
           apply_GBps=round(pr["apply_bytes"] / pr["apply_ms"] / 1e6, 1),
           apply_frac=round(pr["apply_bytes"] / pr["apply_ms"] / 1e6 / hbm, 3),
           fine_post_GBps=round(pr["fine_post_bytes"] / pr["fine_post_ms"] / 1e6, 1),
           japply_GBps=round(pr["japply_bytes"] / pr["japply_ms"] / 1e6, 1), band_ms=round(pr["band_ms"], 3),
           level_nnz=pr["level_nnz"], vcycle_ms=[round(v, 4) for v in pr["vcycle_ms"]])
print(json.dumps(out), flush=True)
b = torch.tensor(np.random.default_rng(42).uniform(-1, 1, J.total_dimension()), device="cuda", dtype=torch.float64)
for orth in ("cgs", "mgs"):
    x, st = api.gmres(op, pc, b, tol=1e-10, max_iter=its, restart=50, scaled=True, orthogonalization=orth)
    out[orth] = dict(gmres_iters=st.iterations, gmres_s=round(st.device_seconds, 3),
                     per_iter_ms=round(st.device_seconds / max(1, st.iterations) * 1e3, 3),
                     final_rel_residual=st.relative_residuals[-1])
    print(json.dumps(out), flush=True)
