"""Live per-level V-cycle times (CUDA graphs, CUDA events) on a BASELINE config.

    python tools/level_profile.py [config] [variant] [ordered|strided]
Level l alone costs vcycle_ms[l] - vcycle_ms[l+1].
"""
import json
import sys

sys.path.insert(0, '.')
from paper_2112_12397_b200 import api  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
var = sys.argv[2] if len(sys.argv) > 2 else "tup"
row_sum = sys.argv[3] if len(sys.argv) > 3 else "ordered"
J = api.Workload(cfg, 42).system()
op = api.BlockSystemOperator(J)
pc = api.GpuPreconditioner.from_host(op, api.HostPreconditioner(J, api.PrecondConfig(
    var, amg=api.AmgConfig(strength_threshold=0.0, row_sum=row_sum))))
p = pc.profile(reps=50)
v = p["vcycle_ms"]
own = [v[l] - (v[l + 1] if l + 1 < len(v) else 0.0) for l in range(len(v))]
print(json.dumps({"config": cfg, "variant": var, "row_sum": row_sum, "apply_ms": round(p["apply_ms"], 4),
                  "japply_ms": round(p["japply_ms"], 4), "levels": p["level_rows"],
                  "vcycle_ms": [round(x, 4) for x in v], "level_own_ms": [round(x, 4) for x in own],
                  "coarse_ms": round(p["coarse_ms"], 4), "band_ms": round(p["band_ms"], 4)}))
