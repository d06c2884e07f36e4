timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
timeout 600 python tools/profile_solve.py 2 tup 500 2>&1 | tail -1
timeout 600 python tools/profile_solve.py 3 tup 100 2>&1 | tail -1
