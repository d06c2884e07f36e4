"""Localize a product-vs-oracle mismatch at a BASELINE config: hierarchy pieces and per-mode applies."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import oracle_lib as O  # noqa: E402
from paper_2112_12397_b200 import api  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
variant = sys.argv[2] if len(sys.argv) > 2 else "tup"
W = api.Workload(cfg, 42)
J = W.system(copy=False)
blocks = [(m.n_rows, m.n_cols, m.row_offsets, m.col_indices, m.values) for m in (J.A, J.C1, J.Q1, J.C2, J.H, J.Q2, J.T, J.F_u)]
osys = O.OracleSystem.from_blocks(J.n_u, J.n_t, J.n_p, blocks)
opc = O.OraclePrecond(osys, variant, coords=J.node_coords, strength_threshold=0.0, row_sum="strided")
hp = api.HostPreconditioner.from_workload(W, api.PrecondConfig(variant, amg=api.AmgConfig(strength_threshold=0.0,
                                                                                           row_sum="strided")))
print("levels", hp.level_sizes(), [opc.level_matrix(l, 0)[0] for l in range(opc.n_levels())])


def same(a, m):
    return (np.array_equal(a[2], m.row_offsets) and np.array_equal(a[3], m.col_indices)
            and np.array_equal(a[4].view(np.uint64), m.values.view(np.uint64)))


for l in range(opc.n_levels()):
    print("A", l, same(opc.level_matrix(l, 0), hp.matrix(0, l)), "diag",
          np.array_equal(opc.level_diag(l), hp.vector(2, l)))
    if l:
        print("P", l, same(opc.level_matrix(l, 1), hp.matrix(1, l)))
print("hblocks", np.array_equal(opc.hblocks(), hp.vector(0)), "vec (T_diag / S_K)", np.array_equal(opc.vec(), hp.vector(1)))
if variant != "tpu":
    print("S2", same(opc.matrix(1), hp.matrix(2)))
op = api.BlockSystemOperator(J)
x = np.random.default_rng(4).uniform(-1, 1, J.total_dimension())
xd = torch.tensor(x, device="cuda", dtype=torch.float64)
for fs in ("sweep", "inverse", "panel"):
    opc.set_factor_solve(fs)
    for rs in ("ordered", "strided"):
        opc.set_row_sum(rs)
        hp.set_upload(rs, fs)
        pc = api.GpuPreconditioner.from_host(op, hp)
        y, ref = pc.apply(xd).cpu().numpy(), opc.apply(x)
        nu, nt = J.n_u, J.n_t
        print(fs, rs, "bitwise", np.array_equal(y, ref), "u", np.array_equal(y[:nu], ref[:nu]), "t",
              np.array_equal(y[nu:nu + nt], ref[nu:nu + nt]), "p", np.array_equal(y[nu + nt:], ref[nu + nt:]), flush=True)
        del pc
