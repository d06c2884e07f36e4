"""Cost probe for parity tests at the large BASELINE configs: generation, product setup + upload, oracle
system / setup, one apply on each side (and whether they agree bitwise), peak RSS.

    python tools/config_costs.py 3 tup
"""
import json
import os
import resource
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle_lib as O  # noqa: E402
from paper_2112_12397_b200 import api  # noqa: E402

cfg = int(sys.argv[1])
variant = sys.argv[2] if len(sys.argv) > 2 else "tup"
out = {"config": cfg, "variant": variant}


def rss():
    return round(resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 1e6, 1)


def lap(key, t0):
    out[key] = round(time.perf_counter() - t0, 2)
    out["rss_GB"] = rss()
    print(json.dumps(out), flush=True)


t0 = time.perf_counter()
W = api.Workload(cfg, 42)
J = W.system(copy=False)
lap("generate_s", t0)
t0 = time.perf_counter()
amg = api.AmgConfig(strength_threshold=0.0, row_sum="strided")
hp = api.HostPreconditioner.from_workload(W, api.PrecondConfig(variant, amg=amg))
lap("host_setup_s", t0)
t0 = time.perf_counter()
op = api.BlockSystemOperator(J)
lap("system_upload_s", t0)
t0 = time.perf_counter()
pc = api.GpuPreconditioner.from_host(op, hp)
lap("precond_upload_s", t0)
out["factor_solve"] = pc.factor_solve
del hp
t0 = time.perf_counter()
blocks = [(m.n_rows, m.n_cols, m.row_offsets, m.col_indices, m.values)
          for m in (J.A, J.C1, J.Q1, J.C2, J.H, J.Q2, J.T, J.F_u)]
osys = O.OracleSystem.from_blocks(J.n_u, J.n_t, J.n_p, blocks)
lap("oracle_system_s", t0)
t0 = time.perf_counter()
opc = O.OraclePrecond(osys, variant, coords=J.node_coords, strength_threshold=0.0, row_sum="strided",
                      factor_solve="sweep")
lap("oracle_setup_s", t0)
x = np.random.default_rng(4).uniform(-1, 1, J.total_dimension())
t0 = time.perf_counter()
ref = opc.apply(x)
lap("oracle_apply_s", t0)
if pc.factor_solve == "inverse":
    t0 = time.perf_counter()
    opc.set_factor_solve("inverse")
    lap("oracle_inverse_build_s", t0)
    t0 = time.perf_counter()
    ref = opc.apply(x)
    lap("oracle_apply_inverse_s", t0)
y = pc.apply(torch.tensor(x, device="cuda", dtype=torch.float64)).cpu().numpy()
out["apply_bitwise"] = bool(np.array_equal(y, ref))
out["apply_rel"] = float(np.linalg.norm(y - ref) / np.linalg.norm(ref))
b = np.random.default_rng(42).uniform(-1, 1, J.total_dimension())
t0 = time.perf_counter()
_, st = O.oracle_gmres(osys, opc, b, tol=1e-10, restart=50, max_iter=3, scaled=True)
lap("oracle_gmres3_s", t0)
print(json.dumps(out), flush=True)
