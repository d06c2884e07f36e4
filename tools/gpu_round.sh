timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
timeout 900 python tools/scale_configs.py 2 3 2>&1 | tail -2 | python -c "
import json,sys
for l in sys.stdin: d=json.loads(l); print({k:d[k] for k in ('config','apply_ms','apply_frac','fine_post_GBps','fine_resid_GBps','japply_GBps','per_iter_ms')})"
