import sys, time, json, numpy as np, torch
sys.path.insert(0,'.')
from paper_2112_12397_b200 import api
cfg = int(sys.argv[1])
W = api.Workload(cfg, 42); J = W.system(); print("system", J.n_u, J.n_t, J.n_p, W.info(), flush=True)
op = api.BlockSystemOperator(J)
b = torch.tensor(np.random.default_rng(42).uniform(-1,1,J.total_dimension()), device="cuda", dtype=torch.float64)
for var in ("tup", "tpu"):
  for th, pre, cyc in ((0.0,1,1), (0.0,2,1), (0.0,1,2), (0.02,1,1), (0.0,3,1)):
    for restart in (50, 200):
        t=time.time(); hp = api.HostPreconditioner(J, api.PrecondConfig(var, amg=api.AmgConfig(strength_threshold=th, pre_sweeps=pre, post_sweeps=pre, cycles_per_apply=cyc))); ts=time.time()-t
        pc = api.GpuPreconditioner.from_host(op, hp)
        x, st = api.gmres(op, pc, b, tol=1e-10, max_iter=500, restart=restart, scaled=True)
        x, st = api.gmres(op, pc, b, tol=1e-10, max_iter=500, restart=restart, scaled=True)
        pr = pc.profile(10)
        print(json.dumps(dict(var=var, th=th, sweeps=pre, cycles=cyc, restart=restart, iters=st.iterations, conv=st.converged, final=st.relative_residuals[-1], solve_s=round(st.device_seconds,4), setup_s=round(ts,2), levels=hp.level_sizes(), apply_ms=round(pr["apply_ms"],3), apply_GBps=round(pr["apply_bytes"]/pr["apply_ms"]/1e6,1), fine_post_GBps=round(pr["fine_post_bytes"]/max(pr["fine_post_ms"],1e-9)/1e6,1), japply_ms=round(pr["japply_ms"],3), band_ms=round(pr["band_ms"],3), coarse_ms=round(pr["coarse_ms"],4))), flush=True)
        del pc, hp
