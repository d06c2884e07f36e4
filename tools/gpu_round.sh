FRACPREC_B200_VERBOSE=1 timeout 900 python tools/setup_time.py 3 2>&1 | grep -v "level start" | head -16
echo ---
FRACPREC_B200_HOST_SETUP=1 FRACPREC_B200_VERBOSE=1 timeout 900 python tools/setup_time.py 3 2>&1 | grep -v "level start" | head -16
