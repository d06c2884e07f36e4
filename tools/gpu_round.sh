timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
timeout 600 python tools/scale_configs.py 2 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:d[k] for k in ('apply_ms','fine_post_GBps','japply_GBps','per_iter_ms')})"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launch_apply_cfg2.csv python tools/profile_apply.py 2 tup 1 > gpurun_out/ncu2.log 2>&1
