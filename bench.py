"""Benchmark of the B200 solve phase (BASELINE.json metric: GMRES + block-AMG solve seconds per system;
preconditioner-apply HBM GB/s vs the HBM peak).

One step = one complete GMRES(50) solve (rtol 1e-10, max 500 iterations) of the driver's block-scaled
system D J D y = b (driver.cpp:229-255) with the t-u-p block preconditioner (inner AMG V-cycle,
weighted Jacobi) on a synthetic BASELINE config, b ~ U[-1,1] seeded.  Default workload: configs[4]
(256x256x128 hex, 40 fractures, 27.6M unknowns), the largest single-GPU config.  The solver options
are the product's defaults — coarse-operator row sums "strided" and classical Gram-Schmidt Arnoldi
(both held to the reference's bars against the reference-order oracle, DESIGN.md §10d/§10e); the
reference's own orders are timed beside it (variants.*_reference_order).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config 1..5]

--impl reference times the CPU oracle (tests/oracle_lib.py: the Eigen-free restatement of the
reference; the reference itself cannot be built here) on this host, on every core, with
the reference's algorithm (ordered row sums, banded sweeps, MGS).  It imports only the workload
generator (workload/) and the oracle, never the B200 package.  Each step is a bounded sample of
GMRES iterations of the same solve; the line reports the measured per-iteration time and the value
per solve = per-iteration time x the solve's iterations (500: the solves on these configs run to
max_iter).
Multi-GPU (torchrun): replicas only — every rank solves its own system, no collective on the data
path.
"""
from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "GMRES+block-AMG solve s/system; precond-apply HBM GB/s vs ~8 TB/s peak"
UNIT = "s/system"
CONFIG_NAMES = {1: "configs[0] 20^3 hex, 1 fracture", 2: "configs[1] 40^3 hex, 1 fracture (lognormal E/aperture)",
                3: "configs[2] 80^3 hex, 3 fractures", 4: "configs[3] 100^3 hex, 10 planes",
                5: "configs[4] 256x256x128 hex, 40 fractures"}


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--variant", default="tup", choices=["tup", "tpu", "tup_star"])
    ap.add_argument("--theta", type=float, default=0.0, help="AMG strength_threshold (amg.hpp:20)")
    ap.add_argument("--factor-solve", default="auto", choices=["auto", "sweep", "inverse", "panel"],
                    help="T / S~2 application (DESIGN.md §5b)")
    ap.add_argument("--restart", type=int, default=50)
    ap.add_argument("--row-sum", default="strided", choices=["ordered", "strided"],
                    help="coarse-operator row-sum order: ordered (the reference's) or strided (32 partials, warp per row)")
    ap.add_argument("--orth", default="cgs", choices=["mgs", "cgs"],
                    help="Arnoldi orthogonalization: mgs (the reference's loop) or cgs (one reduction per pass)")
    ap.add_argument("--tol", type=float, default=1e-10)
    ap.add_argument("--max-iter", type=int, default=500)
    ap.add_argument("--seed", type=int, default=42)
    ap.add_argument("--e2e-steps", type=int, default=5, help="solves timed end to end through the C ABI")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-variants", action="store_true", help="skip the extra variant / config measurements")
    ap.add_argument("--cpu-budget", type=float, default=150.0,
                    help="seconds of oracle GMRES iterations over the whole --impl reference run")
    return ap.parse_args(argv)


# ---- replica bookkeeping (tests/test_replicas.py runs these over gloo, world_size 2)
def replica_seed(base: int, rank: int) -> int:
    """Every rank solves its own system: the workload and rhs seeds are offset by the rank."""
    return base + rank


def replica_max(v: float, ws: int, device: str) -> float:
    """Max over ranks of a per-rank device time (the job is as slow as its slowest replica)."""
    if ws == 1:
        return v
    import torch
    import torch.distributed as dist

    t = torch.tensor([v], device=device, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def whole_job_seconds_per_system(total_s: float, steps: int, ws: int) -> float:
    """ws replicas each solve `steps` systems in total_s (max over ranks): job seconds per system."""
    return total_s / (steps * ws)


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def ncu_traffic(config: int):
    """dram read+write bytes per launch of the roofline kernel from the committed ncu --set full capture."""
    for p in (os.path.join(ROOT, "profiles", "round2", f"ncu_full_cfg{config}.json"),
              os.path.join(ROOT, "profiles", "round1", f"ncu_full_cfg{config}.json")):
        try:
            k = json.load(open(p))["kernels"]["bsr3_EJacobi"]
            return k["dram_bytes_read"] + k["dram_bytes_write"], os.path.relpath(p, ROOT)
        except (OSError, KeyError, ValueError):
            continue
    return None, None


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 200 ms during the timed region."""

    def __init__(self, gpu_index: int):
        self.path = tempfile.mktemp(suffix=".csv")
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.f = open(self.path, "w")
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(gpu_index), f"--query-gpu={q}", "--format=csv,noheader",
                                       "-lms", "200"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self) -> dict:
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.close()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in open(self.path):
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1].split()[0]))
                smax = float(parts[2].split()[0])
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------------------------ reference arm
REFERENCE_ALGORITHM = {"row_sum": "ordered", "factor_solve": "sweep", "orthogonalization": "mgs"}


def run_reference(args) -> dict:
    """The reference's algorithm on the CPU oracle (every host core: threaded row / block loops,
    bitwise the sequential restatement; GMRES dots as fixed-chunk sums), on a bounded sample of GMRES
    iterations of the same solve.  Imports only workload/ and the oracle."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_lib as O
    from workload import gen

    cores = os.cpu_count() or 1
    O.set_threads(cores)
    O.set_chunked_reductions(True)
    t0 = time.perf_counter()
    W = gen.Workload(args.config, args.seed)
    S = W.system(copy=False)
    n = S.total_dimension()
    osys = O.OracleSystem.from_blocks(S.n_u, S.n_t, S.n_p, S.block_list())
    coords = None if S.node_coords is None else S.node_coords.copy()
    del S, W
    gc.collect()
    gen_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    opc = O.OraclePrecond(osys, args.variant, coords=coords, strength_threshold=args.theta,
                          row_sum=REFERENCE_ALGORITHM["row_sum"], factor_solve=REFERENCE_ALGORITHM["factor_solve"])
    setup_s = time.perf_counter() - t0
    b = np.random.default_rng(args.seed).uniform(-1, 1, n)

    def sample(iters):
        t = time.perf_counter()
        _, st = O.oracle_gmres(osys, opc, b, tol=args.tol, restart=args.restart, max_iter=iters, scaled=True)
        return time.perf_counter() - t, st

    # a call of k iterations also pays a fixed part (||b||, the final V y + preconditioner apply and two true
    # residuals); it is measured with k = 0 and taken off, so each step yields the marginal iteration cost
    t_fixed = min(sample(0)[0] for _ in range(2))
    dt, st = sample(1)  # calibration (also warms the caches)
    per_step = args.cpu_budget / max(1, args.steps + args.warmup)
    iters = int(max(1, min(args.restart, per_step / max(dt - t_fixed, 1e-9))))
    for _ in range(args.warmup):
        sample(iters)
    times, its, conv = [], [], False
    for _ in range(args.steps):
        dt, st = sample(iters)
        times.append(dt)
        its.append(st["iterations"])
        conv = conv or st["converged"]
    per_iter = float((np.sum(times) - len(times) * t_fixed) / np.sum(its))
    solve_iters = its[-1] if conv else args.max_iter
    value = per_iter * solve_iters + t_fixed
    sample_txt = (f"{iters} oracle GMRES({args.restart}) iterations per step (Krylov index 0..{iters - 1}); "
                  f"per iteration {per_iter:.3f} s = (step time - {t_fixed:.2f} s fixed part of a call, measured with "
                  f"0 iterations) / iterations; value = per-iteration time x {solve_iters} iterations + the fixed part "
                  f"({'converged' if conv else 'the solve runs to max_iter'}); the MGS cost grows with the Krylov "
                  f"index, so the sample under-counts it (a conservative CPU figure)")
    return {"value": round(value, 4), "per_iteration_s": round(per_iter, 5), "iterations_sampled": int(np.sum(its)),
            "fixed_s": round(t_fixed, 3),
            "steps_s": [round(t, 3) for t in times], "cores": cores, "sample": sample_txt,
            "setup_s": round(setup_s, 1), "generate_s": round(gen_s, 1), "solve_iterations": solve_iters,
            "algorithm": dict(REFERENCE_ALGORITHM, dot_products="fixed 32768-entry chunk sums (threaded)",
                              threads=cores)}


def mapped_product_libraries() -> list:
    """Shared objects of the B200 package mapped into this process (/proc/self/maps)."""
    try:
        maps = open("/proc/self/maps").read().splitlines()
    except OSError:
        return []
    return sorted({ln.split()[-1] for ln in maps if "libfracprec_b200" in ln or "paper_2112_12397_b200" in ln})


def reference_main(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    r = run_reference(args)
    loaded = mapped_product_libraries()
    if loaded:  # the reference arm must not touch the product
        raise SystemExit(f"reference arm mapped the B200 library: {loaded}")
    line = {"impl": "reference", "metric": METRIC, "value": r["value"], "unit": UNIT, "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * float(np.mean(r["steps_s"])), 1),
            "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generator, BASELINE config)",
            "config": {"workload": CONFIG_NAMES[args.config], "variant": args.variant, "gmres": f"GMRES({args.restart})",
                       "rtol": args.tol, "max_iter": args.max_iter, "amg_strength_threshold": args.theta,
                       "smoother": "weighted_jacobi", **r["algorithm"],
                       "deviation_from_ours": "ours runs strided coarse row sums + CGS Arnoldi + its factor "
                                              "application (held to the reference's bars); "
                                              "variants.*_reference_order in our line is the GPU on this algorithm"},
            "per_iteration_s": r["per_iteration_s"], "iterations_sampled": r["iterations_sampled"],
            "cpu_baseline": {"value": r["value"], "unit": UNIT, "cores": r["cores"], "kind": "port",
                             "sample": r["sample"]},
            "e2e": {"value": r["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "setup_s": r["setup_s"], "generate_s": r["generate_s"], "product_libraries_mapped": loaded,
            "note": "the reference (Eigen3/LAPACKE C++) is not buildable here; the oracle restatement is timed"}
    print(json.dumps(line), flush=True)


def cpu_baseline_subprocess(args) -> dict:
    """The reference arm's measurement (a separate process: the oracle's setup needs its own host memory),
    on rank 0 at N = 1, with a shorter budget."""
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", str(args.config),
           "--variant", args.variant, "--steps", "3", "--warmup", "1", "--cpu-budget", "60",
           "--theta", str(args.theta), "--seed", str(args.seed), "--max-iter", str(args.max_iter)]
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    try:
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=1200, env=env)
        line = json.loads(r.stdout.strip().splitlines()[-1])
        c = dict(line["cpu_baseline"])
        c["per_iteration_s"] = line["per_iteration_s"]
        c["setup_s_not_timed"] = line["setup_s"]
        return c
    except Exception as e:  # noqa: BLE001
        return {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
                "sample": f"cpu baseline failed: {type(e).__name__}: {str(e)[:200]}"}


# ------------------------------------------------------------------------------------------ our arm
def solve_fn(api, op, pc, b, x, args, orth=None, probe=False):
    def solve():
        return api.gmres(op, pc, b, tol=args.tol, max_iter=args.max_iter, restart=args.restart, scaled=True, x=x,
                         orthogonalization=orth or args.orth, probe=probe)
    return solve


def timed_variant(api, op, J_or_W, b, flush, args, variant, row_sum, orth, reps=2, from_workload=False,
                  restart=None):
    import torch

    cfg = api.PrecondConfig(variant, amg=api.AmgConfig(strength_threshold=args.theta, row_sum=row_sum),
                            factor_solve=args.factor_solve)
    hp = api.HostPreconditioner.from_workload(J_or_W, cfg) if from_workload else api.HostPreconditioner(J_or_W, cfg)
    pc = api.GpuPreconditioner.from_host(op, hp)
    del hp
    x = torch.empty_like(b)
    if restart is None:
        solve = solve_fn(api, op, pc, b, x, args, orth)
    else:  # full GMRES (restart = max_iter): the reference's own unrestarted semantics (gmres.cpp:24-174)
        def solve():
            return api.gmres(op, pc, b, tol=args.tol, max_iter=args.max_iter, restart=restart, scaled=True, x=x,
                             orthogonalization=orth)
    solve()
    t, st = 0.0, None
    for _ in range(reps):
        flush.zero_()
        torch.cuda.synchronize()
        _, st = solve()
        t += st.device_seconds
    prof = pc.profile(reps=5)
    out = {"s_per_system": round(t / reps, 5), "iterations": st.iterations, "row_sum": row_sum,
           "orthogonalization": orth, "converged": st.converged, "final_rel_residual": st.relative_residuals[-1],
           "factor_solve": pc.factor_solve, "precond_apply_ms": round(prof["apply_ms"], 4),
           "precond_apply_GBps": round(prof["apply_bytes"] / (prof["apply_ms"] * 1e-3) / 1e9, 1)}
    del pc
    return out


def other_variants(api, op, W, b, flush, args) -> dict:
    """The other block preconditioner at the headline config, the reference's summation /
    orthogonalization orders, and configs[1] (the round-1 headline) with every variant."""
    import torch

    out = {}
    other = "tpu" if args.variant != "tpu" else "tup"
    out[f"{other}_cfg{args.config}"] = timed_variant(api, op, W, b, flush, args, other, args.row_sum, args.orth,
                                                      from_workload=True)
    out[f"{args.variant}_cfg{args.config}_reference_order"] = timed_variant(api, op, W, b, flush, args, args.variant,
                                                                            "ordered", "mgs", from_workload=True)
    if args.config != 2:
        W2 = api.Workload(2, args.seed)
        J2 = W2.system(copy=False)
        op2 = api.BlockSystemOperator(J2)
        b2 = torch.tensor(np.random.default_rng(args.seed).uniform(-1, 1, J2.total_dimension()), device="cuda",
                          dtype=torch.float64)
        for v in ("tup", "tpu", "tup_star"):
            out[f"{v}_cfg2"] = timed_variant(api, op2, W2, b2, flush, args, v, args.row_sum, args.orth, reps=3,
                                             from_workload=True)
        out["tup_cfg2_reference_order"] = timed_variant(api, op2, W2, b2, flush, args, "tup", "ordered", "mgs", reps=3,
                                                        from_workload=True)
        # the reference's unrestarted GMRES converges on this workload: time to convergence
        out["tup_cfg2_full_gmres"] = timed_variant(api, op2, W2, b2, flush, args, "tup", args.row_sum, args.orth,
                                                   reps=3, from_workload=True, restart=args.max_iter)
    return out


def run_ours(args):
    import torch

    ws, rank, local = dist_env()
    if ws > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    torch.cuda.set_device(local)
    from paper_2112_12397_b200 import api

    seed = replica_seed(args.seed, rank)  # replicas: independent systems
    # Replicas share one host: the generated system (config 5: ~30 GB per rank) and the setup's host
    # phases are built one rank at a time, and a replica drops its host copy once it is on the device
    # (the extra variants, which rebuild from it, are N = 1 only).
    if ws > 1:
        args.no_variants = True
    for turn in range(ws):
        if turn == rank:
            t0 = time.perf_counter()
            W = api.Workload(args.config, seed)
            J = W.system(copy=False)
            gen_s = time.perf_counter() - t0
            t0 = time.perf_counter()
            op = api.BlockSystemOperator(J)
            upload_s = time.perf_counter() - t0
            t0 = time.perf_counter()
            cfg = api.PrecondConfig(args.variant, amg=api.AmgConfig(strength_threshold=args.theta, row_sum=args.row_sum),
                                    factor_solve=args.factor_solve)
            hp = api.HostPreconditioner.from_workload(W, cfg)
            setup_s = time.perf_counter() - t0
            t0 = time.perf_counter()
            pc = api.GpuPreconditioner.from_host(op, hp)
            levels = hp.level_sizes()
            del hp
            precond_upload_s = time.perf_counter() - t0
            n = J.total_dimension()
            n_u, n_t, n_p = J.n_u, J.n_t, J.n_p
            if ws > 1:
                J = W = None
                gc.collect()
        if ws > 1:
            import torch.distributed as dist

            dist.barrier()
    b_host = np.random.default_rng(seed).uniform(-1, 1, n)
    b = torch.tensor(b_host, device="cuda", dtype=torch.float64)
    x = torch.empty_like(b)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")  # 256 MB > 126 MB L2
    # probe: CUDA events around the roofline kernel inside every 8th step's graph (roofline.achieved)
    solve = solve_fn(api, op, pc, b, x, args, probe=True)
    warmup = max(3, args.warmup)
    for _ in range(warmup):
        _, st = solve()

    def barrier():
        if ws > 1:
            import torch.distributed as dist

            dist.barrier()
        torch.cuda.synchronize()

    clocks = ClockSampler(local)
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    stats, launches = [], 0
    ev0.record()
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()  # flush complete before the solve (the solver's stream is non-blocking)
        _, st = solve()
        stats.append(st)
        launches += st.kernel_launches
    ev1.record()
    barrier()
    clk = clocks.stop()
    # device time of the solves, from CUDA events the solver records on its own (launching) stream
    # around each solve (fp_solve_stats.device_seconds); the torch-stream bracket is a cross-check
    dev_s = sum(st_.device_seconds for st_ in stats)
    bracket_ms = ev0.elapsed_time(ev1)
    total_s = replica_max(dev_s, ws, "cuda")
    value = whole_job_seconds_per_system(total_s, args.steps, ws)

    # e2e: the C ABI with pinned host buffers; H2D of b and D2H of x inside the timed region
    b_pin = torch.tensor(b_host, dtype=torch.float64).pin_memory()
    x_pin = torch.empty(n, dtype=torch.float64).pin_memory()

    def solve_host():
        return api.gmres(op, pc, b_pin.numpy(), tol=args.tol, max_iter=args.max_iter, restart=args.restart,
                         scaled=True, x=x_pin.numpy(), orthogonalization=args.orth)

    e2e_steps = max(1, min(args.steps, args.e2e_steps))
    barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        flush.zero_()
        torch.cuda.synchronize()
        solve_host()
    barrier()
    e2e_s = replica_max(time.perf_counter() - t0, ws, "cuda")
    e2e_value = e2e_s / (e2e_steps * ws)

    prof = pc.profile(reps=20)
    hbm, peak_src = peaks()
    # dominant kernel: the finest-level BSR3 Jacobi sweep (4 per t-u-p apply); its average duration
    # over the timed solves, from the CUDA events bracketing it in every 8th step's graph
    probe_ms = sum(st_.probe_ms for st_ in stats)
    probe_n = sum(st_.probe_launches for st_ in stats)
    fine_ms = probe_ms / probe_n if probe_n else prof["fine_post_ms"]
    fine_gbs = prof["fine_post_bytes"] / (fine_ms * 1e-3) / 1e9 if fine_ms else None
    apply_gbs = prof["apply_bytes"] / (prof["apply_ms"] * 1e-3) / 1e9
    traffic, traffic_src = ncu_traffic(args.config)
    st = stats[-1]
    line = None
    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 6), "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": warmup, "ms_per_step": round(total_s / args.steps * 1e3, 3), "higher_is_better": False,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded generator, BASELINE config)",
            "config": {"workload": CONFIG_NAMES[args.config], "n_u": n_u, "n_t": n_t, "n_p": n_p,
                       "unknowns": n, "variant": args.variant, "gmres": f"GMRES({args.restart})", "rtol": args.tol,
                       "max_iter": args.max_iter, "orthogonalization": args.orth, "row_sum": args.row_sum,
                       "amg_strength_threshold": args.theta, "smoother": "weighted_jacobi",
                       "factor_solve": pc.factor_solve,
                       "l2": "256 MB buffer written between timed solves; working set > 126 MB L2",
                       "parallelism": f"replicas x{ws}" if ws > 1 else "single GPU"},
            "iterations": st.iterations, "converged": st.converged, "restarts": st.restarts,
            "reorth_steps": st.reorth_steps,
            "final_rel_residual": st.relative_residuals[-1] if st.relative_residuals else None,
            "e2e": {"value": round(e2e_value, 6), "unit": UNIT, "h2d_bytes_per_step": 8 * n, "d2h_bytes_per_step": 8 * n,
                    "steps": e2e_steps, "path": "fp_gmres through the C ABI, pinned host b / x"},
            "roofline": {"bound": "hbm", "kernel": "bsr3 Jacobi post-smoothing sweep, finest AMG level (S1)",
                         "achieved": round(fine_gbs, 1) if fine_gbs else None, "peak": hbm, "unit": "GB/s",
                         "frac": round(fine_gbs / hbm, 3) if fine_gbs else None, "traffic": traffic,
                         "traffic_source": traffic_src, "peak_source": peak_src,
                         "algorithmic_bytes_per_launch": prof["fine_post_bytes"],
                         "avg_launch_ms": round(fine_ms, 4), "launches_timed": probe_n,
                         "timing": "CUDA events around the kernel inside every 8th Arnoldi step's graph, over the timed region",
                         "isolated_loop_ms": round(prof["fine_post_ms"], 4)},
            "precond_apply": {"GBps": round(apply_gbs, 1), "frac": round(apply_gbs / hbm, 3),
                              "ms": round(prof["apply_ms"], 4), "algorithmic_bytes": prof["apply_bytes"],
                              "wasted_bytes": prof["apply_wasted_bytes"], "kernels": prof["apply_launches"],
                              "ledger": "SURVEY §8(d): each stored operator once per use, B_factor = 12 (nnz(L) + nnz(U)); "
                                        "bytes streamed beyond that (explicit block inverses) are wasted_bytes"},
            "profile_ms": {k: round(prof[k], 4) for k in ("apply_ms", "japply_ms", "fine_resid_ms", "fine_post_ms",
                                                          "band_ms", "coarse_ms")},
            "amg_levels": prof["level_rows"], "amg_level_nnz": prof["level_nnz"], "setup_levels": levels,
            "gpu_launches": int(launches),
            "timing": "value = CUDA events on the solver's stream around each solve (max over ranks); "
                      f"torch-stream bracket incl. L2 flush: {bracket_ms / args.steps:.3f} ms per step",
            "clocks": clk, "generate_s": round(gen_s, 2), "system_upload_s": round(upload_s, 2),
            "setup_s": round(setup_s, 2), "precond_upload_s": round(precond_upload_s, 2),
        }
    del J, pc, solve, solve_host
    gc.collect()
    torch.cuda.empty_cache()  # the variants build their own preconditioners (config 5: ~70 GB each)
    if rank == 0 and not args.no_variants:
        line["variants"] = other_variants(api, op, W, b, flush, args)
    del W, op
    gc.collect()
    torch.cuda.empty_cache()
    if rank == 0 and not args.no_cpu_baseline and ws == 1:
        line["cpu_baseline"] = cpu_baseline_subprocess(args)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        reference_main(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
