"""The oracle's threaded loops (oracle/par.hpp) change nothing: setup, applies and GMRES on several
threads are bitwise the single-threaded restatement (the reference's own order).  CPU only."""
import numpy as np
import pytest

import oracle_lib as O
import contextlib
from workload import gen


@pytest.fixture(scope="module")
def config1():
    W = gen.Workload(1, 42)  # BASELINE configs[0]: 30,466 unknowns, A with 2.07M entries
    S = W.system()
    return S, O.OracleSystem.from_blocks(S.n_u, S.n_t, S.n_p, S.block_list())


@contextlib.contextmanager
def threads(n):
    old = O.threads()
    O.set_threads(n)
    try:
        yield
    finally:
        O.set_threads(old)


def build(osys, S, variant, n_threads, **kw):
    with threads(n_threads):
        return O.OraclePrecond(osys, variant, coords=S.node_coords, strength_threshold=0.0, **kw)


def same_csr(a, b):
    return a[0] == b[0] and a[1] == b[1] and all(np.array_equal(x, y) for x, y in zip(a[2:], b[2:]))


@pytest.mark.parametrize("variant", ["tpu", "tup"])
def test_threaded_setup_and_apply_are_bitwise_sequential(config1, variant):
    S, osys = config1
    seq = build(osys, S, variant, 1)
    par = build(osys, S, variant, 8)
    assert seq.n_levels() == par.n_levels() >= 3
    for l in range(seq.n_levels()):
        for which in (0, 1) if l else (0,):
            assert same_csr(seq.level_matrix(l, which), par.level_matrix(l, which)), (l, which)
        assert np.array_equal(seq.level_diag(l), par.level_diag(l))
    assert same_csr(seq.matrix(1), par.matrix(1)) if variant == "tup" else True
    x = np.random.default_rng(2).uniform(-1, 1, osys.n)
    ref = seq.apply(x)
    for row_sum in ("ordered", "strided"):
        seq.set_row_sum(row_sum)
        par.set_row_sum(row_sum)
        with threads(1):
            ref = seq.apply(x)
        with threads(8):
            assert np.array_equal(par.apply(x), ref), row_sum
            assert np.array_equal(seq.apply(x), ref), row_sum  # the same handle, threaded apply


def test_threaded_gmres_history_is_bitwise_sequential(config1):
    S, osys = config1
    pc = build(osys, S, "tup", 1)
    b = np.random.default_rng(42).uniform(-1, 1, osys.n)
    with threads(1):
        x1, st1 = O.oracle_gmres(osys, pc, b, tol=1e-10, restart=50, max_iter=40, scaled=True)
    with threads(8):
        x8, st8 = O.oracle_gmres(osys, pc, b, tol=1e-10, restart=50, max_iter=40, scaled=True)
    assert st1["iterations"] == st8["iterations"]
    assert np.array_equal(st1["history"], st8["history"])
    assert np.array_equal(x1, x8)


def test_threaded_transpose_and_factor_inverse(config1):
    S, osys = config1
    # the system's block apply runs the threaded spmv; the inverse build threads over columns
    x = np.random.default_rng(4).uniform(-1, 1, osys.n)
    with threads(1):
        y1 = osys.apply(x)
        pc1 = O.OraclePrecond(osys, "tup", coords=S.node_coords, strength_threshold=0.0, factor_solve="inverse")
        z1 = pc1.apply(x)
    with threads(8):
        y8 = osys.apply(x)
        pc8 = O.OraclePrecond(osys, "tup", coords=S.node_coords, strength_threshold=0.0, factor_solve="inverse")
        z8 = pc8.apply(x)
    assert np.array_equal(y1, y8)
    assert np.array_equal(z1, z8)


def test_chunked_reductions_stay_within_the_reference_bars(config1):
    """The chunk-sum dot option (large-config tests, bench CPU legs) is a rounding change only."""
    S, osys = config1
    pc = build(osys, S, "tup", 8)
    b = np.random.default_rng(42).uniform(-1, 1, osys.n)
    with threads(8):
        x1, st1 = O.oracle_gmres(osys, pc, b, tol=1e-10, restart=50, max_iter=500, scaled=True)
        O.set_chunked_reductions(True)
        try:
            x2, st2 = O.oracle_gmres(osys, pc, b, tol=1e-10, restart=50, max_iter=500, scaled=True)
        finally:
            O.set_chunked_reductions(False)
    assert st1["converged"] and st2["converged"]
    assert abs(st1["iterations"] - st2["iterations"]) <= 2
    assert np.linalg.norm(x1 - x2) <= 1e-8 * np.linalg.norm(x1)
