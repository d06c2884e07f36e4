"""The oracle against the reference's own known-answer tests.

The reference ships no golden vectors and cannot be built here (Eigen3,
LAPACKE, doctest and CLI11 are absent), so the oracle is pinned by every
known-answer test and property the reference suite holds for the solve path
(tests/unit/test_csr.cpp, test_gmres.cpp, test_amg.cpp, test_precond.cpp and the
SPEC.md examples), re-expressed in oracle/kat.cpp on the reference's own seeded
fixtures (test_helpers.hpp).
"""
import os
import subprocess

import oracle_lib

EXPECTED = [
    "spmv identity and zero", "spmv dense row-by-row oracle", "spmv_transpose examples",
    "spmv_transpose equals spmv of transpose", "spgemm examples and dense oracle", "spgemm associativity",
    "add_scaled union pattern", "bdiag3_extract slices diagonal blocks", "bdiag3_solve identity, scaling and dense oracle",
    "diag_extract", "restrict_submatrix gathers dense blocks", "csr invariants validated",
    "gmres on identity converges in one iteration", "gmres with exact inverse preconditioner: one iteration",
    "gmres 2x2 direct-solve oracle", "gmres monotone residuals and finite termination",
    "right preconditioning: Arnoldi estimate equals true residual", "gmres basis orthogonality after reorthogonalization",
    "gmres reports non-convergence at max_iter", "gmres happy breakdown yields exact solve",
    "amg single level below max_coarse is a direct solve", "amg 1d poisson coarsening rate near one third",
    "amg galerkin identity on every level", "amg apply is linear (sgs)", "amg apply is linear (jacobi)",
    "amg v-cycle is symmetric for symmetric input with sgs", "amg 1d poisson error propagation spectral radius",
    "amg rigid body modes reproduced per aggregate", "amg h-scalability on 3d poisson (sgs)",
    "amg h-scalability on 3d poisson (jacobi)", "amg rejects zero diagonal and non-square input",
    "tpu decoupled: S == A, apply splits per physics", "tpu all-stick schur complement is symmetric",
    "tpu mixed-state schur matches dense triple product",
    "tup build: stick -> S_K = 0, decoupled -> S1 == A, mixed -> dense S1",
    "fixed_stress_diag matches dense restriction oracle", "tpu pressure unit vectors are fixed points",
    "apply_tpu equals the dense block-LDU factor product", "apply_tup and tup_star equal their dense factor forms",
    "tup_star equals tup on decoupled input and w = 0 maps to 0", "inner-solver cost contract: 1 tpu, 2 tup, 1 tup_star",
    "preconditioner applications are linear (amg sgs)", "preconditioner applications are linear (amg jacobi)",
]


def test_oracle_known_answer_suite():
    if not os.path.exists(oracle_lib.KAT):
        oracle_lib.build()
    r = subprocess.run([oracle_lib.KAT], capture_output=True, text=True, timeout=600)
    passed = {ln[5:] for ln in r.stdout.splitlines() if ln.startswith("PASS ")}
    failed = [ln for ln in r.stdout.splitlines() if ln.startswith("FAIL ")]
    assert not failed, "\n".join(failed)
    assert r.returncode == 0, r.stdout[-2000:]
    missing = [t for t in EXPECTED if t not in passed]
    assert not missing, missing
