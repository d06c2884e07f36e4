"""Drive every kernel family of the solve path once on small inputs, for compute-sanitizer
(memcheck / racecheck / synccheck):

    compute-sanitizer --tool memcheck python tools/sanitize.py

Covers: the system upload and device layouts (BSR3, SELL, node-blocked, windowed pipeline, R = P^T),
the device setup (SpGEMM incl. the block-per-row path, strength graph, transpose), the preconditioner
applies (t-p-u, t-u-p, t-u-p*; ordered / strided rows incl. the quad-per-row layout; sweep / inverse / panel factor; Jacobi,
Chebyshev, multicolour GS), the cooperative MGS / CGS Arnoldi kernels with the one-ahead step and a
mid-cycle restage (restart 120), the large-n orthogonalization chain, and the fracture-block assembly.
Prints one line per phase; exits non-zero on any CUDA error.
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2112_12397_b200 import api  # noqa: E402


def say(msg):
    print(f"[sanitize] {msg}", flush=True)


def run_case(J, variant, row_sum, factor, smoother="weighted_jacobi", theta=0.0):
    op = api.BlockSystemOperator(J)
    amg = api.AmgConfig(strength_threshold=theta, row_sum=row_sum, smoother=smoother)
    try:
        pc = api.GpuPreconditioner.from_host(
            op, api.HostPreconditioner(J, api.PrecondConfig(variant, amg=amg, factor_solve=factor)))
    except ValueError as e:  # panel mode on a pivoting factor
        say(f"skip {variant} {row_sum} {factor} {smoother}: {e}")
        return
    x = torch.tensor(np.random.default_rng(1).uniform(-1, 1, J.total_dimension()), device="cuda", dtype=torch.float64)
    pc.apply(x)
    op.apply(x)
    torch.cuda.synchronize()
    say(f"apply {variant} {row_sum} {factor} {smoother}: ok")


def main():
    spec = dict(cells=(8, 6, 6), fractures=[(0, 0.25, 0.0, 1.0, 0.0, 1.0), (0, 0.75, 0.0, 1.0, 0.5, 1.0)],
                frac_stick=0.5, frac_slip=0.3, E_sigma_ln=0.5, aperture_sigma_ln=0.3)
    W = api.Workload(spec=spec, seed=3)
    J = W.system()
    for variant in ("tpu", "tup", "tup_star"):
        for row_sum in ("ordered", "strided"):
            for factor in ("sweep", "inverse", "panel"):
                run_case(J, variant, row_sum, factor)
    for smoother in ("chebyshev", "multicolor_gs"):
        run_case(J, "tup", "strided", "auto", smoother)
    # theta = 0.08 on config 1: the dense level-2 Galerkin product (block-per-row SpGEMM)
    J1 = api.Workload(1, 42).system()
    run_case(J1, "tup", "ordered", "auto", theta=0.08)
    # config 2: the windowed pipeline (level-1 operator >= 2048 rows, ordered) and node-blocked P_1
    os.environ["FRACPREC_B200_BP3_MIN_NODES"] = "1000"
    J2 = api.Workload(2, 42).system()
    run_case(J2, "tup", "ordered", "auto")
    # the quad-per-row strided layout forced onto every coarse operator (shared column lists, sorted slices)
    os.environ["FRACPREC_B200_SRT_MIN_ROWS"] = "1"
    run_case(J2, "tup", "strided", "auto")
    run_case(J, "tpu", "strided", "auto")
    del os.environ["FRACPREC_B200_SRT_MIN_ROWS"]
    op = api.BlockSystemOperator(J2)
    pc = api.GpuPreconditioner.from_host(op, api.HostPreconditioner(J2, api.PrecondConfig(
        "tup", amg=api.AmgConfig(strength_threshold=0.0, row_sum="strided"))))
    b = torch.tensor(np.random.default_rng(42).uniform(-1, 1, J2.total_dimension()), device="cuda", dtype=torch.float64)
    for orth in ("mgs", "cgs"):
        for restart in (50, 120):  # restart 120: mid-cycle true-residual checks with a step in flight
            _, st = api.gmres(op, pc, b, tol=1e-10, max_iter=130, restart=restart, scaled=True, orthogonalization=orth)
            say(f"gmres {orth} restart {restart}: {st.iterations} iterations")
    os.environ["FRACPREC_B200_WIDE_ORTH"] = "1"  # the large-n orthogonalization chain on a small system
    op2 = api.BlockSystemOperator(J)
    pc2 = api.GpuPreconditioner.from_host(op2, api.HostPreconditioner(J, api.PrecondConfig("tup")))
    bb = np.random.default_rng(2).uniform(-1, 1, J.total_dimension())
    for orth in ("mgs", "cgs"):
        _, st = api.gmres(op2, pc2, bb, tol=1e-10, max_iter=60, restart=50, scaled=True, orthogonalization=orth)
        say(f"gmres wide {orth}: {st.iterations} iterations")
    # fracture-block assembly on the device, installed into the system
    FA = api.FractureAssembly(W)
    FA.run(W.state(), api.BlockSystemOperator(J))
    torch.cuda.synchronize()
    say("fracture assembly: ok")
    say("done")


if __name__ == "__main__":
    main()
