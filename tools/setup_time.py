"""Host setup time of a BASELINE config (lean path), with the setup's SpGEMMs on the device or the host.

    python tools/setup_time.py 2          # FRACPREC_B200_HOST_SETUP=1 forces the host SpGEMM
"""
import sys
import time

sys.path.insert(0, ".")
from paper_2112_12397_b200 import api  # noqa: E402

cfg = int(sys.argv[1])
W = api.Workload(cfg, 42)
t0 = time.perf_counter()
hp = api.HostPreconditioner.from_workload(W, api.PrecondConfig("tup", amg=api.AmgConfig(strength_threshold=0.0)))
print(f"config {cfg}: setup {time.perf_counter() - t0:.2f} s, spgemm backend {api.setup_backend()}, "
      f"levels {hp.level_sizes()}", flush=True)
