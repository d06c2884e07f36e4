"""C-ABI library checks that need no GPU: it loads, exports every symbol the
headers declare, validates arguments like the reference (std::invalid_argument
-> FP_INVALID_ARGUMENT), and its host-side setup (build_tpu / build_tup,
amg_setup) reproduces the oracle's bit for bit."""
import ctypes as C
import glob
import os
import re

import numpy as np
import pytest

import oracle_lib as O
from paper_2112_12397_b200 import _native as N
from paper_2112_12397_b200 import api

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols(header: str):
    txt = open(os.path.join(ROOT, "include", header)).read()
    return set(re.findall(r"^[A-Za-z_][\w \*]*?\b(fp_\w+)\s*\(", txt, flags=re.M))


def test_library_exports_every_declared_symbol():
    """include/fracprec_b200.h -> libfracprec_b200.so; include/fracprec_workload.h -> the generator's
    libfp_workload.so, which does not pull in the solve library."""
    from workload import gen

    names = declared_symbols("fracprec_b200.h")
    assert len(names) >= 25
    lib = C.CDLL(N.LIB_PATH)
    missing = [n for n in sorted(names) if not hasattr(lib, n)]
    assert not missing, missing
    assert set(N.SIGNATURES) == names, set(N.SIGNATURES) ^ names
    assert b"sm_100a" in N.lib.fp_version()
    wnames = declared_symbols("fracprec_workload.h")
    assert set(gen.SIGNATURES) == wnames, set(gen.SIGNATURES) ^ wnames
    wl = C.CDLL(gen.LIB_PATH)
    assert not [n for n in sorted(wnames) if not hasattr(wl, n)]
    import subprocess

    r = subprocess.run(["ldd", gen.LIB_PATH], capture_output=True, text=True)
    assert "fracprec_b200" not in r.stdout and "libcuda" not in r.stdout, r.stdout


def test_shared_library_is_sm100a_only():
    import subprocess

    r = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", N.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in r.stdout
    assert "sm_90" not in r.stdout and "sm_80" not in r.stdout


def csr(rows, cols, trips):
    rp = np.zeros(rows + 1, np.int64)
    trips = sorted(trips)
    for r, _, _ in trips:
        rp[r + 1] += 1
    return api.CsrMatrix(rows, cols, np.cumsum(rp), np.array([c for _, c, _ in trips], np.int32),
                         np.array([v for _, _, v in trips]))


def test_invalid_arguments_are_reported_not_thrown():
    A = csr(3, 3, [(0, 0, 1.0), (1, 1, 1.0), (2, 2, 1.0)])
    Z = api.CsrMatrix.empty
    # n_t != 3 n_p (block.cpp:49-52)
    J = api.BlockSystem(3, 2, 1, A, Z(3, 2), Z(3, 1), Z(2, 3), Z(2, 2), Z(1, 3), csr(1, 1, [(0, 0, 1.0)]))
    h = C.c_void_p()
    st = N.lib.fp_system_create(C.byref(J.view()), C.byref(h))
    assert st == N.FP_INVALID_ARGUMENT and b"n_t must equal 3*n_p" in N.lib.fp_last_error()
    # unsorted columns (csr.cpp:31-47 invariants)
    bad = api.CsrMatrix(2, 2, np.array([0, 2, 2]), np.array([1, 0], np.int32), np.array([1.0, 1.0]))
    J2 = api.BlockSystem(2, 0, 0, bad, Z(2, 0), Z(2, 0), Z(0, 2), Z(0, 0), Z(0, 2), Z(0, 0))
    assert N.lib.fp_system_create(C.byref(J2.view()), C.byref(h)) == N.FP_INVALID_ARGUMENT
    assert b"strictly increasing" in N.lib.fp_last_error()
    # wrong shapes in the host builder
    with pytest.raises(ValueError):
        api.HostPreconditioner(J, api.PrecondConfig("tup"))
    with pytest.raises(ValueError):
        api.PrecondConfig("tpu", inner="direct").native()


def test_new_options_are_validated():
    """row_sum / orthogonalization: unknown values are rejected at the API and at the ABI."""
    J = small_workload(seed=7)
    with pytest.raises(ValueError, match="row_sum"):
        api.AmgConfig(row_sum="pairwise").native()
    c = api.AmgConfig().native()
    c.row_sum = 7
    cfg = N.FpPrecondConfig()
    cfg.variant, cfg.amg, cfg.factor_solve = 1, c, 0
    h = C.c_void_p()
    st = N.lib.fp_host_precond_build(C.byref(J.view()), C.byref(cfg), None, 0, C.byref(h))
    assert st == N.FP_INVALID_ARGUMENT and b"row_sum" in N.lib.fp_last_error()
    # defaults are the reference's orders
    d = N.FpAmgConfig()
    N.lib.fp_amg_config_default(C.byref(d))
    assert d.row_sum == 0 and api.AmgConfig().row_sum == "ordered"
    assert N.FpGmresOptions().orthogonalization == 0


def test_zero_diagonal_is_a_numerical_error():
    # amg_setup rejects a zero diagonal with numerical_error (amg.cpp:205-207)
    n_u, n_p = 6, 1
    trips = [(i, i, 2.0) for i in range(n_u) if i != 4] + [(4, 3, 1.0), (3, 4, 1.0)]
    A = csr(n_u, n_u, trips)
    Z = api.CsrMatrix.empty
    H = csr(3, 3, [(0, 0, 1.0), (1, 1, 1.0), (2, 2, 1.0)])
    J = api.BlockSystem(n_u, 3, n_p, A, Z(n_u, 3), Z(n_u, 1), Z(3, n_u), H, Z(1, n_u), csr(1, 1, [(0, 0, 1.0)]))
    with pytest.raises(N.NumericalError, match="zero diagonal"):
        api.HostPreconditioner(J, api.PrecondConfig("tup", amg=api.AmgConfig(max_coarse=2)))


def small_workload(seed=7, cells=(6, 6, 6), fracs=((0, 0.5, 0.0, 1.0, 0.0, 1.0),), **kw):
    spec = dict(cells=cells, fractures=list(fracs), frac_stick=0.5, frac_slip=0.3, E_sigma_ln=0.5,
                aperture_sigma_ln=0.3, **kw)
    return api.Workload(spec=spec, seed=seed).system()


def oracle_system(J):
    blocks = [(m.n_rows, m.n_cols, m.row_offsets, m.col_indices, m.values)
              for m in (J.A, J.C1, J.Q1, J.C2, J.H, J.Q2, J.T, J.F_u)]
    return O.OracleSystem.from_blocks(J.n_u, J.n_t, J.n_p, blocks)


def same_csr(a, m: api.CsrMatrix):
    return (a[0] == m.n_rows and np.array_equal(a[2], m.row_offsets) and np.array_equal(a[3], m.col_indices)
            and np.array_equal(a[4], m.values))


@pytest.mark.parametrize("variant", ["tpu", "tup"])
def test_host_setup_is_bitwise_the_oracle_setup(variant):
    J = small_workload()
    osys = oracle_system(J)
    opc = O.OraclePrecond(osys, variant, coords=J.node_coords)
    hp = api.HostPreconditioner(J, api.PrecondConfig(variant))
    assert hp.level_sizes() == [opc.level_matrix(l, 0)[0] for l in range(opc.n_levels())]
    for l in range(opc.n_levels()):
        assert same_csr(opc.level_matrix(l, 0), hp.matrix(0, l)), f"A_{l}"
        assert np.array_equal(opc.level_diag(l), hp.vector(2, l))
        if l > 0:
            assert same_csr(opc.level_matrix(l, 1), hp.matrix(1, l)), f"P_{l}"
    assert np.array_equal(opc.hblocks(), hp.vector(0))
    assert np.array_equal(opc.vec(), hp.vector(1))  # T_diag (tpu) / S_K (tup)
    if variant == "tup":
        assert same_csr(opc.matrix(1), hp.matrix(2))  # S~2


def test_workload_sizes_follow_the_reference_mesh_rules():
    # config 1 has 9261 + 19*19 duplicated nodes -> n_u = 28,866; nnz(A) = 2,074,086
    J = api.Workload(1, 42).system()
    assert (J.n_u, J.n_t, J.n_p) == (28866, 1200, 400)
    assert J.A.nnz == 2074086
    assert J.node_coords.shape == (9622, 3)
    # the duplicated fracture nodes sit on the fracture plane x = 0.5
    assert np.all(J.node_coords[9261:, 0] == 0.5)


def test_workload_custom_mesh_counts():
    # 4x4x2 box with a 2x2-face fracture (the reference's small_spec, test_model.cpp:22-32 geometry)
    spec = dict(cells=(4, 4, 2), length=(4.0, 4.0, 2.0), fractures=[(0, 2.0, 1.0, 3.0, 0.0, 2.0)])
    J = api.Workload(spec=spec, seed=1).system()
    # nodes 5*5*3 = 75, interior patch nodes (jb in (1,3), jc in (0,2)) = 1*1 -> 1 duplicate
    assert J.n_u == 3 * 76 and J.n_p == 4 and J.n_t == 12
    with pytest.raises(ValueError, match="not grid aligned"):
        api.Workload(spec=dict(cells=(2, 2, 2), fractures=[(0, 0.3, 0.0, 1.0, 0.0, 1.0)]), seed=1)


@pytest.mark.parametrize("variant", ["tpu", "tup", "tup_star"])
def test_oracle_block_inverse_is_the_sweep_operator(variant):
    """factor_solve = inverse applies the same operator as the
    reference's SparseFactor sweeps, up to rounding (1e-12 relative, the apply bar)."""
    J = small_workload(seed=41, cells=(8, 6, 6), fracs=((0, 0.25, 0.0, 1.0, 0.0, 1.0), (0, 0.75, 0.0, 1.0, 0.5, 1.0)))
    osys = oracle_system(J)
    opc = O.OraclePrecond(osys, variant, coords=J.node_coords)
    rng = np.random.default_rng(6)
    xs = rng.uniform(-1, 1, (3, J.total_dimension()))
    ref = [opc.apply(x) for x in xs]
    opc.set_factor_solve("inverse")
    for x, r in zip(xs, ref):
        y = opc.apply(x)
        assert np.linalg.norm(y - r) <= 1e-12 * np.linalg.norm(r)
    opc.set_factor_solve("sweep")
    assert all(np.array_equal(opc.apply(x), r) for x, r in zip(xs, ref))


@pytest.mark.parametrize("case", ["2frac", "config1"])
@pytest.mark.parametrize("variant", ["tpu", "tup", "tup_star"])
def test_oracle_panel_solve_is_the_sweep_operator(variant, case):
    """factor_solve = panel: the block-bidiagonal panel form of the same banded factor
    applies the sweeps' operator up to rounding (1e-12 relative, the apply bar)."""
    if case == "config1":
        J = api.Workload(1, 42).system()
    else:
        J = small_workload(seed=41, cells=(8, 6, 6), fracs=((0, 0.25, 0.0, 1.0, 0.0, 1.0), (0, 0.75, 0.0, 1.0, 0.5, 1.0)))
    osys = oracle_system(J)
    opc = O.OraclePrecond(osys, variant, coords=J.node_coords, strength_threshold=0.0)
    assert not opc.factor_pivots()  # T (LDL^T) and the workloads' S~2 factor without interchanges
    rng = np.random.default_rng(7)
    xs = rng.uniform(-1, 1, (3, J.total_dimension()))
    ref = [opc.apply(x) for x in xs]
    opc.set_factor_solve("panel")
    for x, r in zip(xs, ref):
        y = opc.apply(x)
        assert np.linalg.norm(y - r) <= 1e-12 * np.linalg.norm(r), np.linalg.norm(y - r) / np.linalg.norm(r)
    opc.set_factor_solve("sweep")
    assert all(np.array_equal(opc.apply(x), r) for x, r in zip(xs, ref))


@pytest.mark.parametrize("theta", [0.08, 0.0])
@pytest.mark.parametrize("variant", ["tpu", "tup", "tup_star"])
def test_oracle_strided_row_sums_are_the_ordered_operator(variant, theta):
    """row_sum = strided only regroups the coarse operators' row sums:
    the preconditioner applies the reference-order operator to within the 1e-12 bar."""
    J = small_workload(seed=43, cells=(8, 8, 8), fracs=((0, 0.25, 0.0, 1.0, 0.0, 1.0), (0, 0.75, 0.0, 1.0, 0.5, 1.0)))
    osys = oracle_system(J)
    opc = O.OraclePrecond(osys, variant, coords=J.node_coords, strength_threshold=theta)
    assert opc.n_levels() >= 3
    rng = np.random.default_rng(8)
    xs = rng.uniform(-1, 1, (3, J.total_dimension()))
    ref = [opc.apply(x) for x in xs]
    opc.set_row_sum("strided")
    diff = [np.linalg.norm(opc.apply(x) - r) / np.linalg.norm(r) for x, r in zip(xs, ref)]
    assert max(diff) <= 1e-12, diff
    assert max(diff) > 0.0  # the order does change the rounding
    opc.set_row_sum("ordered")
    assert all(np.array_equal(opc.apply(x), r) for x, r in zip(xs, ref))


def test_oracle_strided_gmres_within_reference_bars():
    J = small_workload(seed=23, cells=(8, 8, 6))
    osys = oracle_system(J)
    b = np.random.default_rng(42).uniform(-1, 1, J.total_dimension())
    ref = O.OraclePrecond(osys, "tup", coords=J.node_coords)
    x_ref, st_ref = O.oracle_gmres(osys, ref, b, tol=1e-10, restart=50, max_iter=300, scaled=True)
    strided = O.OraclePrecond(osys, "tup", coords=J.node_coords, row_sum="strided")
    x, st = O.oracle_gmres(osys, strided, b, tol=1e-10, restart=50, max_iter=300, scaled=True)
    assert st_ref["converged"] and st["converged"]
    assert abs(st["iterations"] - st_ref["iterations"]) <= 2
    assert np.linalg.norm(x - x_ref) <= 1e-8 * np.linalg.norm(x_ref)


def test_factor_solve_is_validated():
    with pytest.raises(ValueError, match="factor_solve"):
        api.PrecondConfig(factor_solve="cholesky").native()
    J = small_workload()
    cfg = api.PrecondConfig("tup").native()
    cfg.factor_solve = 7
    h = C.c_void_p()
    st = N.lib.fp_host_precond_build(C.byref(J.view()), C.byref(cfg), None, 0, C.byref(h))
    assert st == N.FP_INVALID_ARGUMENT and b"factor_solve" in N.lib.fp_last_error()


@pytest.mark.parametrize("variant", ["tpu", "tup"])
def test_chebyshev_setup_is_bitwise_the_oracle(variant):
    """Chebyshev smoother (extension): the host's power-iteration lambda_max
    per level equals the oracle's bit for bit, and brackets rho(D^-1 A) from above."""
    J = small_workload(seed=43)
    amg = dict(smoother=2, chebyshev_degree=3, chebyshev_ratio=20.0, power_iterations=12)
    opc = O.OraclePrecond(osys := oracle_system(J), variant, coords=J.node_coords, **amg)
    hp = api.HostPreconditioner(J, api.PrecondConfig(variant, amg=api.AmgConfig(
        smoother="chebyshev", chebyshev_degree=3, chebyshev_ratio=20.0, power_iterations=12)))
    nl = opc.n_levels()
    assert hp.level_sizes() == [opc.level_matrix(l, 0)[0] for l in range(nl)]
    for l in range(nl - 1):
        lam = hp.vector(3, l)[0]
        assert lam == opc.level_lambda(l) and lam > 0
        r, c, rp, ci, v = opc.level_matrix(l, 0)
        if r <= 1500:  # dense check of the estimate on the small levels
            A = np.zeros((r, c))
            A[np.repeat(np.arange(r), np.diff(rp)), ci] = v
            rho = max(abs(np.linalg.eigvals(A / np.diag(A)[:, None])))
            assert rho * 0.8 < lam < rho * 1.1 * (1 + 1e-9)
    del osys


def test_oracle_chebyshev_vcycle_contracts():
    """The restated Chebyshev V-cycle is a convergent stationary iteration on the inner operator."""
    J = small_workload(seed=44)
    osys = oracle_system(J)
    rho = {}
    for sm in (0, 2):  # weighted Jacobi (reference option) vs Chebyshev degree 2, ratio 10
        opc = O.OraclePrecond(osys, "tup", coords=J.node_coords, smoother=sm, chebyshev_degree=2)
        r, c, rp, ci, v = opc.level_matrix(0, 0)
        A = np.zeros((r, c))
        A[np.repeat(np.arange(r), np.diff(rp)), ci] = v
        B = np.column_stack([opc.amg_apply(e) for e in np.eye(r)])  # B ~ A^-1
        rho[sm] = max(abs(np.linalg.eigvals(np.eye(r) - B @ A)))
    assert rho[2] < 0.6 and rho[2] < rho[0], rho  # measured: 0.49 vs 1.06


def test_oracle_multicolor_gs_vcycle_contracts():
    """The multicolour symmetric Gauss-Seidel smoother (extension): rows of one
    colour never couple, and its V-cycle contracts like the reference's lexicographic SGS (and better
    than weighted Jacobi) on the inner operator."""
    J = small_workload(seed=44)
    osys = oracle_system(J)
    rho = {}
    for sm in (0, 1, 3):  # weighted Jacobi, lexicographic SGS (reference default), multicolour SGS
        opc = O.OraclePrecond(osys, "tup", coords=J.node_coords, smoother=sm)
        r, c, rp, ci, v = opc.level_matrix(0, 0)
        A = np.zeros((r, c))
        A[np.repeat(np.arange(r), np.diff(rp)), ci] = v
        if sm == 3:
            rows, off = opc.level_colors(0)
            color = np.empty(r, np.int64)
            for k in range(len(off) - 1):
                color[rows[off[k]:off[k + 1]]] = k
            row_of = np.repeat(np.arange(r), np.diff(rp))
            off_diag = row_of != ci
            assert not np.any(color[row_of[off_diag]] == color[ci[off_diag]])
        B = np.column_stack([opc.amg_apply(e) for e in np.eye(r)])  # B ~ A^-1
        rho[sm] = max(abs(np.linalg.eigvals(np.eye(r) - B @ A)))
    assert rho[3] < 0.5 and rho[3] < rho[0], rho


@pytest.mark.parametrize("name,cells,length,fracs,expect", [
    # test_model.cpp:93-100: the trivial 2^3 cube (27 nodes, no fracture)
    ("cube", (2, 2, 2), (1.0, 1.0, 1.0), [], (81, 0, 0)),
    # test_model.cpp:102-105, presets.cpp test1: x 10 cells, y segments 8/20/8 cells, z 6 cells, the patch
    # at x = 5 over y cells 8..28 and the full z; the counts depend on the cell topology only, so the y axis is
    # written with one unit per cell (ticks 8 and 28 exact)
    ("test1", (10, 36, 6), (10.0, 36.0, 6.0), [(0, 5.0, 8.0, 28.0, 0.0, 6.0)], (8832, 360, 120)),
    # test_model.cpp:107-110, presets.cpp make_test2a(25): four x-planes over [0.2, 0.8]^2
    ("test2a-coarse", (25, 25, 25), (1.0, 1.0, 1.0), [(0, x, 0.2, 0.8, 0.2, 0.8) for x in (0.2, 0.4, 0.6, 0.8)],
     (55080, 2700, 900)),
    # test_model.cpp:112-121, presets.cpp make_test2b(level): nine x-planes over [0.2, 0.8]^2
    ("test2b-1", (10, 10, 10), (1.0, 1.0, 1.0), [(0, 0.1 * i, 0.2, 0.8, 0.2, 0.8) for i in range(1, 10)],
     (4668, 972, 324)),
    ("test2b-2", (20, 20, 20), (1.0, 1.0, 1.0), [(0, 0.1 * i, 0.2, 0.8, 0.2, 0.8) for i in range(1, 10)],
     (31050, 3888, 1296)),
])
def test_reference_mesh_count_pins(name, cells, length, fracs, expect):
    """The reference's own mesh pins (/root/reference/proj/tests/unit/test_model.cpp:93-129) re-expressed
    against the generator that feeds every parity test (workload/workload.cpp restating mesh.cpp's
    fracture-node duplication): n_u, n_t, n_p and n_t = 3 n_p."""
    from workload import gen

    S = gen.Workload(spec=dict(cells=cells, length=length, fractures=fracs), seed=1).system(copy=False)
    assert (S.n_u, S.n_t, S.n_p) == expect
    assert S.n_t == 3 * S.n_p
