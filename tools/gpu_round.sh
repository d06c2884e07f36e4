timeout 1500 python tools/smoother_compare.py 2 2>&1 | tail -8
