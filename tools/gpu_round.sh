mkdir -p gpurun_out
grep -E "MemTotal|MemAvailable" /proc/meminfo; nproc
avail_gb=$(awk '/MemAvailable/ {print int($2/1000/1000)}' /proc/meminfo)
limit=$(( avail_gb - 20 ))
echo "limit ${limit} GB"
FRACPREC_B200_VERBOSE=1 LIMIT_GB=$limit timeout 2700 tools/watchdog.sh python tools/big_config.py 5 30 > gpurun_out/big5.json 2> gpurun_out/big5.err
echo "rc=$?"
tail -1 gpurun_out/big5.json; grep -E "watchdog|rss" gpurun_out/big5.err | tail -12
