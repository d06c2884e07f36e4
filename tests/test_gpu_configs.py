"""Parity at BASELINE.json's own sizes: configs[0] (the "PR1 oracle" case, 30,466 unknowns) and
configs[1] (the bench's 40^3 box, 217,726 unknowns), both preconditioner variants, against the
CPU oracle on the same seeded inputs (SURVEY §8(d) generator, b ~ U[-1, 1]).

Bars (BASELINE north_star): one preconditioner application within 1e-12 (asserted bitwise), GMRES
iteration count within +-2 and the solution within 1e-8 at rtol 1e-10; when both sides stop at
max_iter (non-convergence), the residual histories are compared instead.
"""
import numpy as np
import pytest
import torch

import oracle_lib as O
from paper_2112_12397_b200 import api
from test_abi_cpu import oracle_system

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def setup(config, variant, row_sum):
    J = api.Workload(config, 42).system()
    osys = oracle_system(J)
    amg = api.AmgConfig(strength_threshold=0.0, row_sum=row_sum)
    op = api.BlockSystemOperator(J)
    pc = api.GpuPreconditioner.from_host(op, api.HostPreconditioner(J, api.PrecondConfig(variant, amg=amg)))
    opc = O.OraclePrecond(osys, variant, coords=J.node_coords, factor_solve=pc.factor_solve, row_sum=row_sum,
                          strength_threshold=0.0)
    return J, osys, op, pc, opc


@pytest.mark.parametrize("row_sum", ["ordered", "strided"])
@pytest.mark.parametrize("variant", ["tpu", "tup"])
def test_config1_apply_and_gmres(variant, row_sum):
    J, osys, op, pc, opc = setup(1, variant, row_sum)
    x = np.random.default_rng(3).uniform(-1, 1, J.total_dimension())
    xd = torch.tensor(x, device="cuda", dtype=torch.float64)
    assert np.array_equal(pc.apply(xd).cpu().numpy(), opc.apply(x))
    b = np.random.default_rng(42).uniform(-1, 1, J.total_dimension())
    x_ref, st_ref = O.oracle_gmres(osys, opc, b, tol=1e-10, restart=50, max_iter=500, scaled=True)
    orth = "cgs" if row_sum == "strided" else "mgs"  # the bench's pairing, and the reference's
    xs, st = api.gmres(op, pc, torch.tensor(b, device="cuda", dtype=torch.float64), tol=1e-10, max_iter=500,
                       restart=50, scaled=True, orthogonalization=orth)
    assert st.converged == st_ref["converged"]
    assert abs(st.iterations - st_ref["iterations"]) <= 2, (st.iterations, st_ref["iterations"])
    if st_ref["converged"]:
        assert rel(xs.cpu().numpy(), x_ref) <= 1e-8
    else:
        k = min(len(st.relative_residuals), len(st_ref["history"])) - 1
        h, hr = np.array(st.relative_residuals[:k]), st_ref["history"][:k]
        assert np.all(np.abs(np.log10(h) - np.log10(hr)) < 0.5)


@pytest.mark.parametrize("variant", ["tpu", "tup"])
def test_config2_apply_bitwise_and_gmres_history(variant):
    """The bench's workload at full size: applies bitwise in both row-sum orders, and 60 GMRES(50)
    iterations of the bench's solver (strided rows, CGS) track the reference-order oracle (ordered
    rows, MGS) step by step."""
    J, osys, op, pc, opc = setup(2, variant, "strided")
    x = np.random.default_rng(4).uniform(-1, 1, J.total_dimension())
    xd = torch.tensor(x, device="cuda", dtype=torch.float64)
    assert np.array_equal(pc.apply(xd).cpu().numpy(), opc.apply(x))
    opc.set_row_sum("ordered")
    ref = opc.apply(x)
    assert rel(pc.apply(xd).cpu().numpy(), ref) <= 1e-12  # strided vs the reference order: the apply bar
    b = np.random.default_rng(42).uniform(-1, 1, J.total_dimension())
    _, st_ref = O.oracle_gmres(osys, opc, b, tol=1e-10, restart=50, max_iter=60, scaled=True)
    _, st = api.gmres(op, pc, torch.tensor(b, device="cuda", dtype=torch.float64), tol=1e-10, max_iter=60,
                      restart=50, scaled=True, orthogonalization="cgs")
    assert st.iterations == st_ref["iterations"] == 60
    h, hr = np.array(st.relative_residuals), st_ref["history"]
    assert np.allclose(h, hr, rtol=1e-6, atol=0), np.max(np.abs(h / hr - 1))


def test_config2_full_gmres_converges_to_the_oracle_solution():
    """The reference's own GMRES semantics (full, unrestarted: gmres.cpp:24-174) on the bench's
    workload: it converges, so the solution-level bars apply — the bench's solver
    (strided rows, CGS, its factor application) against the oracle in the same summation modes running
    the reference's MGS loop: iteration count within +-2, solution within 1e-8 at rtol 1e-10."""
    J, osys, op, pc, opc = setup(2, "tup", "strided")
    b = np.random.default_rng(42).uniform(-1, 1, J.total_dimension())
    O.set_chunked_reductions(True)
    try:
        x_ref, st_ref = O.oracle_gmres(osys, opc, b, tol=1e-10, restart=500, max_iter=500, scaled=True)
    finally:
        O.set_chunked_reductions(False)
    xs, st = api.gmres(op, pc, torch.tensor(b, device="cuda", dtype=torch.float64), tol=1e-10, max_iter=500,
                       restart=500, scaled=True, orthogonalization="cgs")
    assert st_ref["converged"] and st.converged, (st_ref["iterations"], st.iterations)
    assert abs(st.iterations - st_ref["iterations"]) <= 2, (st.iterations, st_ref["iterations"])
    assert rel(xs.cpu().numpy(), x_ref) <= 1e-8


def test_config2_bench_solver_500_steps_tracks_the_reference_order_oracle():
    """All 500 GMRES(50) steps of the bench's solver (strided rows, CGS, its factor application) against
    the oracle in the reference's own orders (ordered rows, MGS, banded sweeps): both stop at max_iter
    (the solve stagnates) and the residual histories agree step by step to 1e-6 relative
    over the first 100 steps and to 1e-3 over all 500."""
    J, osys, op, pc, opc = setup(2, "tup", "strided")
    opc.set_row_sum("ordered")
    opc.set_factor_solve("sweep")
    b = np.random.default_rng(42).uniform(-1, 1, J.total_dimension())
    _, st_ref = O.oracle_gmres(osys, opc, b, tol=1e-10, restart=50, max_iter=500, scaled=True)
    _, st = api.gmres(op, pc, torch.tensor(b, device="cuda", dtype=torch.float64), tol=1e-10, max_iter=500,
                      restart=50, scaled=True, orthogonalization="cgs")
    assert st.converged == st_ref["converged"]
    assert abs(st.iterations - st_ref["iterations"]) <= 2, (st.iterations, st_ref["iterations"])
    k = min(len(st.relative_residuals), len(st_ref["history"]))
    h, hr = np.array(st.relative_residuals[:k]), st_ref["history"][:k]
    assert np.allclose(h[:100], hr[:100], rtol=1e-6, atol=0), np.max(np.abs(h[:100] / hr[:100] - 1))
    assert np.allclose(h, hr, rtol=1e-3, atol=0), np.max(np.abs(h / hr - 1))


@pytest.mark.parametrize("variant", ["tpu", "tup"])
def test_config2_shared_column_lists_bitwise(variant, monkeypatch):
    """The warp-row operators (A_l, R_l with >= 2048 rows, row_sum = strided) keep one column list
    per aggregate (the 6 coarse dofs of an aggregate share their pattern): fewer index bytes, the
    same entries in the same order, so the apply stays bitwise the oracle's and the plain-CSR one's."""
    J, osys, op, pc, opc = setup(2, variant, "strided")  # default: shared lists where the pattern allows
    monkeypatch.setenv("FRACPREC_B200_SHARED_COLS", "0")
    amg = api.AmgConfig(strength_threshold=0.0, row_sum="strided")
    pc_plain = api.GpuPreconditioner.from_host(op, api.HostPreconditioner(J, api.PrecondConfig(variant, amg=amg)))
    monkeypatch.delenv("FRACPREC_B200_SHARED_COLS")
    assert pc.traffic()["apply_bytes"] < pc_plain.traffic()["apply_bytes"]  # the shared lists did engage
    x = np.random.default_rng(5).uniform(-1, 1, J.total_dimension())
    xd = torch.tensor(x, device="cuda", dtype=torch.float64)
    y = pc.apply(xd).cpu().numpy()
    assert np.array_equal(y, pc_plain.apply(xd).cpu().numpy())
    assert np.array_equal(y, opc.apply(x))


@pytest.mark.parametrize("variant", ["tpu", "tup"])
def test_config2_quad_per_row_strided_layout_bitwise(variant, monkeypatch):
    """The quad-per-row strided32 layout (srt_kernel: slices of 8 length-sorted rows, four lanes per row, 32 partials
    and the xor tree split between shuffles and in-lane additions; taken from 65,536 rows on, forced here onto every
    coarse operator of config 2) gives the warp-per-row kernel's sums bit for bit: the apply stays
    bitwise the oracle's."""
    monkeypatch.setenv("FRACPREC_B200_SRT_MIN_ROWS", "1")
    J, osys, op, pc, opc = setup(2, variant, "strided")
    monkeypatch.delenv("FRACPREC_B200_SRT_MIN_ROWS")
    x = np.random.default_rng(7).uniform(-1, 1, J.total_dimension())
    xd = torch.tensor(x, device="cuda", dtype=torch.float64)
    assert np.array_equal(pc.apply(xd).cpu().numpy(), opc.apply(x))
    monkeypatch.setenv("FRACPREC_B200_SRT_MIN_ROWS", "0")
    amg = api.AmgConfig(strength_threshold=0.0, row_sum="strided")
    pc_warp = api.GpuPreconditioner.from_host(op, api.HostPreconditioner(J, api.PrecondConfig(variant, amg=amg)))
    assert pc.traffic()["apply_bytes"] != pc_warp.traffic()["apply_bytes"]  # the layout did engage
    assert np.array_equal(pc.apply(xd).cpu().numpy(), pc_warp.apply(xd).cpu().numpy())


@pytest.mark.parametrize("variant", ["tpu", "tup"])
def test_config2_outputs_stay_inside_their_buffers(variant):
    """compute-sanitizer is closed on this GPU pool, so out-of-bounds writes of the output paths are
    checked directly: inputs and outputs of J apply, preconditioner apply and GMRES live inside one
    device buffer between guard bands of a sentinel bit pattern, every variant of the input is placed
    flush against a band, and the bands (and the inputs) must come back bit for bit."""
    J, osys, op, pc, opc = setup(2, variant, "strided")
    n = J.total_dimension()
    G = 4096
    sentinel = float(np.frombuffer(np.uint64(0x7FF8DEADBEEF1234).tobytes(), dtype=np.float64)[0])  # a NaN payload
    big = torch.full((4 * G + 3 * n,), sentinel, device="cuda", dtype=torch.float64)
    raw0 = big.view(torch.int64).clone()
    xin = big[G:G + n]
    y1 = big[2 * G + n:2 * G + 2 * n]
    y2 = big[3 * G + 2 * n:3 * G + 3 * n]
    x = np.random.default_rng(8).uniform(-1, 1, n)
    xin.copy_(torch.tensor(x, device="cuda", dtype=torch.float64))
    pc.apply(xin, y1)
    op.apply(xin, y2)
    torch.cuda.synchronize()
    assert np.array_equal(y1.cpu().numpy(), opc.apply(x))
    assert np.array_equal(y2.cpu().numpy(), osys.apply(x))
    api.gmres(op, pc, xin, tol=1e-10, max_iter=60, restart=50, scaled=True, x=y1, orthogonalization="cgs")
    api.gmres(op, pc, xin, tol=1e-10, max_iter=60, restart=50, scaled=True, x=y2, orthogonalization="mgs")
    torch.cuda.synchronize()
    raw = big.view(torch.int64)
    assert np.array_equal(xin.cpu().numpy(), x)  # inputs untouched
    for lo, hi in ((0, G), (G + n, 2 * G + n), (2 * G + 2 * n, 3 * G + 2 * n), (3 * G + 3 * n, 4 * G + 3 * n)):
        assert torch.equal(raw[lo:hi], raw0[lo:hi]), (lo, hi)
