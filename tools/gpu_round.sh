timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 600 python tools/profile_solve.py 2 tup 500 2>&1 | tail -1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_solve_cfg2.csv python tools/profile_solve.py 2 tup 50 > gpurun_out/ncus.log 2>&1
