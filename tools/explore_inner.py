"""Exploration: does a much stronger inner AMG (more sweeps / cycles) make config 2 converge?"""
import json, sys, time
import numpy as np, torch
sys.path.insert(0, '.')
from paper_2112_12397_b200 import api
def run(J, tag, var, th, pre, cyc, restart=50, maxit=500):
    op = api.BlockSystemOperator(J)
    b = torch.tensor(np.random.default_rng(42).uniform(-1, 1, J.total_dimension()), device="cuda", dtype=torch.float64)
    hp = api.HostPreconditioner(J, api.PrecondConfig(var, amg=api.AmgConfig(strength_threshold=th, pre_sweeps=pre, post_sweeps=pre, cycles_per_apply=cyc)))
    pc = api.GpuPreconditioner.from_host(op, hp)
    x, st = api.gmres(op, pc, b, tol=1e-10, max_iter=maxit, restart=restart, scaled=True)
    pr = pc.profile(5)
    print(json.dumps(dict(tag=tag, var=var, th=th, sweeps=pre, cycles=cyc, restart=restart, iters=st.iterations, conv=st.converged,
                          final=st.relative_residuals[-1], solve_s=round(st.device_seconds, 3), levels=pr["level_rows"], level_nnz=pr["level_nnz"],
                          apply_ms=round(pr["apply_ms"], 3))), flush=True)
J2 = api.Workload(2, 42).system()
for pre, cyc in ((1, 1), (5, 1), (3, 3), (8, 2)):
    run(J2, "cfg2", "tup", 0.0, pre, cyc)
hom = dict(cells=(40, 40, 40), fractures=[(0, 0.5, 0, 1, 0, 1)], frac_stick=0.6, frac_slip=0.3, E_sigma_ln=0.0, aperture_sigma_ln=0.3)
Jh = api.Workload(spec=hom, seed=42).system()
run(Jh, "40^3 homogeneous E", "tup", 0.0, 1, 1)
run(Jh, "40^3 homogeneous E", "tup", 0.0, 3, 3)
stick = dict(hom, E_sigma_ln=0.5, frac_stick=1.0, frac_slip=0.0)
Js = api.Workload(spec=stick, seed=42).system()
run(Js, "40^3 lognormal E, all stick", "tup", 0.0, 1, 1)
run(Js, "40^3 lognormal E, all stick", "tup", 0.0, 3, 3)
