"""A/B of upload-time format switches on one BASELINE config: the system and the preconditioner setup are built once,
then the preconditioner is uploaded and profiled once per environment setting.

    python tools/ab_formats.py 5 "" FRACPREC_B200_WARP_PF=0 FRACPREC_B200_SHARED_COLS=0,FRACPREC_B200_WARP_PF=0
Each argument after the config is a comma-separated list of VAR=value (empty string = defaults).
"""
import gc
import json
import os
import sys

import torch

sys.path.insert(0, ".")
from paper_2112_12397_b200 import api  # noqa: E402

cfg = int(sys.argv[1])
settings = sys.argv[2:] or [""]
variant = os.environ.get("AB_VARIANT", "tup")
W = api.Workload(cfg, 42)
J = W.system(copy=False)
hp = api.HostPreconditioner.from_workload(W, api.PrecondConfig(variant, amg=api.AmgConfig(strength_threshold=0.0,
                                                                                          row_sum=os.environ.get("AB_ROW_SUM", "strided"))))
op = api.BlockSystemOperator(J)
for st in settings:
    kv = [x.split("=", 1) for x in st.split(",") if x]
    for k, v in kv:
        os.environ[k] = v
    pc = api.GpuPreconditioner.from_host(op, hp)
    pr = pc.profile(5)
    out = {"config": cfg, "setting": st or "defaults", "apply_ms": round(pr["apply_ms"], 4),
           "apply_GB": round(pr["apply_bytes"] / 1e9, 3), "apply_GBps": round(pr["apply_bytes"] / pr["apply_ms"] / 1e6, 1),
           "band_ms": round(pr["band_ms"], 4), "vcycle_ms": [round(x, 4) for x in pr["vcycle_ms"]],
           "fine_post_ms": round(pr["fine_post_ms"], 4)}
    print(json.dumps(out), flush=True)
    for k, _ in kv:
        del os.environ[k]
    del pc
    gc.collect()
    torch.cuda.empty_cache()
