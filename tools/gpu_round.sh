timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k gmres 2>&1 | tail -1
for g in 148 96 64 32; do echo "grid $g"; FRACPREC_B200_MGS_GRID=$g timeout 600 python tools/profile_solve.py 2 tup 200 2>&1 | tail -1; done
