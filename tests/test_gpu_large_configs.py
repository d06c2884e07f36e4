"""Parity at BASELINE.json's large configs (north_star: "5-30M-unknown configs"):
configs[2] (80^3, 3 fractures, 1.73M unknowns), configs[3] (100^3, 10 planes, 3.78M) and
configs[4] (256x256x128, 40 fractures, 27.6M; one apply per variant), both preconditioner variants, GPU (product-built
hierarchy, uploaded) against the CPU oracle (its own setup, on every host core; oracle/par.hpp) on
the same seeded inputs.

Bars: one preconditioner application bitwise (so within 1e-12) in both coarse row-sum orders and
both factor applications; GMRES(50) over >= 100 iterations (both sides run the same steps: the
solves stagnate) with the iteration count within +-2 and the relative-residual history
matched step by step.  conftest.py runs this module first so `-x` cannot hide it behind a slower
failure.  Config 5's oracle setup peaks near 170 GB of host memory (the product's device setup and
upload finish and free their host data first).
"""
import gc
import os
import time

import numpy as np
import pytest
import torch

import oracle_lib as O
from paper_2112_12397_b200 import api

pytestmark = [pytest.mark.gpu, pytest.mark.large]

GMRES_STEPS = 100


def log(msg):
    print(f"[large-configs {time.strftime('%H:%M:%S')}] {msg}", flush=True)


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def host_precond(W, variant):
    cfg = api.PrecondConfig(variant, amg=api.AmgConfig(strength_threshold=0.0, row_sum="strided"))
    return api.HostPreconditioner.from_workload(W, cfg)


def gpu_precond(hp, op, row_sum, factor_solve):
    hp.set_upload(row_sum, factor_solve)
    return api.GpuPreconditioner.from_host(op, hp)


def oracle_for(J, variant):
    blocks = [(m.n_rows, m.n_cols, m.row_offsets, m.col_indices, m.values)
              for m in (J.A, J.C1, J.Q1, J.C2, J.H, J.Q2, J.T, J.F_u)]
    osys = O.OracleSystem.from_blocks(J.n_u, J.n_t, J.n_p, blocks)
    opc = O.OraclePrecond(osys, variant, coords=J.node_coords, strength_threshold=0.0, row_sum="strided")
    return osys, opc


@pytest.mark.parametrize("variant", ["tup", "tpu"])
@pytest.mark.parametrize("config", [3, 4])
def test_large_config_apply_bitwise_and_gmres_history(config, variant):
    t0 = time.perf_counter()
    W = api.Workload(config, 42)
    J = W.system(copy=False)
    n = J.total_dimension()
    op = api.BlockSystemOperator(J)
    osys, opc = oracle_for(J, variant)
    log(f"config {config} {variant}: n={n}, oracle setup done at {time.perf_counter() - t0:.0f} s")
    hp = host_precond(W, variant)
    log(f"config {config} {variant}: product setup done at {time.perf_counter() - t0:.0f} s")
    x = np.random.default_rng(4).uniform(-1, 1, n)
    xd = torch.tensor(x, device="cuda", dtype=torch.float64)
    for factor_solve in ("sweep", "inverse", "panel"):
        opc.set_factor_solve(factor_solve)
        for row_sum in ("ordered", "strided"):
            pc = gpu_precond(hp, op, row_sum, factor_solve)
            assert pc.factor_solve == factor_solve
            opc.set_row_sum(row_sum)
            y, ref = pc.apply(xd).cpu().numpy(), opc.apply(x)
            assert np.array_equal(y, ref), (factor_solve, row_sum, rel(y, ref))
            if (factor_solve, row_sum) != ("panel", "strided"):
                del pc
                gc.collect()
    del hp
    gc.collect()
    log(f"config {config} {variant}: applies bitwise at {time.perf_counter() - t0:.0f} s")
    # GMRES(50): the bench's solver (strided rows, CGS, panel factor) against the oracle in the same
    # summation modes running the reference's MGS loop
    b = np.random.default_rng(42).uniform(-1, 1, n)
    _, st = api.gmres(op, pc, torch.tensor(b, device="cuda", dtype=torch.float64), tol=1e-10,
                      max_iter=GMRES_STEPS, restart=50, scaled=True, orthogonalization="cgs")
    O.set_chunked_reductions(True)  # threaded chunk-sum dots (bitwise-sequential dots take ~1 s per step here)
    try:
        _, st_ref = O.oracle_gmres(osys, opc, b, tol=1e-10, restart=50, max_iter=GMRES_STEPS, scaled=True)
    finally:
        O.set_chunked_reductions(False)
    log(f"config {config} {variant}: GMRES {st.iterations} / {st_ref['iterations']} iterations, final "
        f"{st.relative_residuals[-1]:.3e} / {st_ref['history'][-1]:.3e} at {time.perf_counter() - t0:.0f} s")
    assert st.converged == st_ref["converged"]
    assert abs(st.iterations - st_ref["iterations"]) <= 2, (st.iterations, st_ref["iterations"])
    k = min(len(st.relative_residuals), len(st_ref["history"]))
    assert k >= min(GMRES_STEPS, st_ref["iterations"]) - 2
    h, hr = np.array(st.relative_residuals[:k]), st_ref["history"][:k]
    assert np.allclose(h, hr, rtol=1e-6, atol=0), np.max(np.abs(h / hr - 1))


CONFIG5_VARIANTS = os.environ.get("FRACPREC_CONFIG5_VARIANTS", "tup").split(",")


@pytest.mark.skipif(os.environ.get("FRACPREC_SKIP_CONFIG5") == "1", reason="FRACPREC_SKIP_CONFIG5=1")
@pytest.mark.parametrize("variant", CONFIG5_VARIANTS)
def test_config5_apply_bitwise(variant):
    """configs[4] at full size (27.6M unknowns, A with 2.1e9 entries, int64 offsets): one application,
    GPU (product-built hierarchy) bitwise the oracle's (oracle-built hierarchy).  t-u-p (the bench's
    variant) by default; FRACPREC_CONFIG5_VARIANTS=tpu runs t-p-u — one variant per pytest process,
    since the oracle's setup peaks near 170 GB of host memory and two back to back do not fit in one
    process on a 196 GB box (profiles/round2/config5_tpu_bitwise.log is that run)."""
    t0 = time.perf_counter()
    W = api.Workload(5, 42)
    J = W.system(copy=False)
    n = J.total_dimension()
    op = api.BlockSystemOperator(J)
    hp = host_precond(W, variant)
    pc = gpu_precond(hp, op, "strided", "auto")
    del hp
    gc.collect()
    x = np.random.default_rng(5).uniform(-1, 1, n)
    y = pc.apply(torch.tensor(x, device="cuda", dtype=torch.float64)).cpu().numpy()
    factor_solve = pc.factor_solve
    del pc, op
    gc.collect()
    torch.cuda.empty_cache()
    log(f"config 5 {variant}: GPU apply done at {time.perf_counter() - t0:.0f} s ({factor_solve})")
    osys, opc = oracle_for(J, variant)
    del J, W
    gc.collect()
    opc.set_factor_solve(factor_solve)
    ref = opc.apply(x)
    log(f"config 5 {variant}: oracle apply done at {time.perf_counter() - t0:.0f} s")
    assert np.array_equal(y, ref), rel(y, ref)
