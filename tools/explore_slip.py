"""Exploration: outer GMRES(50) convergence vs the synthetic slip-increment magnitude and state mix (40^3)."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
from paper_2112_12397_b200 import api  # noqa: E402


def run(spec, tag, var="tup", th=0.0, pre=1, cyc=1, restart=50, maxit=500):
    J = api.Workload(spec=spec, seed=42).system()
    op = api.BlockSystemOperator(J)
    b = torch.tensor(np.random.default_rng(42).uniform(-1, 1, J.total_dimension()), device="cuda", dtype=torch.float64)
    hp = api.HostPreconditioner(J, api.PrecondConfig(var, amg=api.AmgConfig(strength_threshold=th, pre_sweeps=pre,
                                                                           post_sweeps=pre, cycles_per_apply=cyc)))
    pc = api.GpuPreconditioner.from_host(op, hp)
    x, st = api.gmres(op, pc, b, tol=1e-10, max_iter=maxit, restart=restart, scaled=True)
    print(json.dumps(dict(tag=tag, var=var, sweeps=pre, cycles=cyc, restart=restart, iters=st.iterations,
                          conv=st.converged, final=st.relative_residuals[-1], solve_s=round(st.device_seconds, 3))),
          flush=True)


base = dict(cells=(40, 40, 40), fractures=[(0, 0.5, 0, 1, 0, 1)], frac_stick=0.6, frac_slip=0.3, E_sigma_ln=0.5,
            aperture_sigma_ln=0.3)
for sf in (10.0, 100.0, 1e4):
    run(dict(base, slip_factor=sf), f"slip_factor={sf}")
    run(dict(base, slip_factor=sf), f"slip_factor={sf}", var="tpu")
run(dict(base, frac_stick=0.9, frac_slip=0.0), "stick 90 / open 10")
run(dict(base, frac_stick=0.7, frac_slip=0.3), "stick 70 / slip 30, no open")
run(dict(base, slip_factor=1e4), "slip_factor=1e4 strong inner", pre=3, cyc=2)
