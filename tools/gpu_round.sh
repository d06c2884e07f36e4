for c in 2 3 4; do timeout 900 python tools/setup_time.py $c 2>&1 | tail -1; done
FRACPREC_B200_VERBOSE=1 timeout 900 python tools/setup_time.py 3 2>&1 | grep -v "level start" | head -9
