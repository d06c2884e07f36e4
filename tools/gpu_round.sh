timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 900 python tools/scale_configs.py 2 3 2>&1 | tail -2 | cut -c1-600
FRACPREC_B200_NO_PDL=1 timeout 900 python tools/scale_configs.py 2 2>&1 | tail -1 | cut -c1-600
timeout 600 python tools/profile_solve.py 2 tup 500 2>&1 | tail -1
FRACPREC_B200_NO_PDL=1 timeout 600 python tools/profile_solve.py 2 tup 500 2>&1 | tail -1
