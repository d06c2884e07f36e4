#!/bin/bash
# Run a command, killing it (by its exact PID) if its resident memory exceeds LIMIT_GB.
#   LIMIT_GB=170 tools/watchdog.sh python tools/big_config.py 5
LIMIT_KB=$(( ${LIMIT_GB:-170} * 1000 * 1000 ))
"$@" &
pid=$!
peak=0
while kill -0 "$pid" 2>/dev/null; do
  rss=$(awk '/VmRSS/ {print $2}' /proc/$pid/status 2>/dev/null || echo 0)
  rss=${rss:-0}
  [ "$rss" -gt "$peak" ] && peak=$rss
  if [ "$rss" -gt "$LIMIT_KB" ]; then
    echo "watchdog: RSS ${rss} kB > ${LIMIT_KB} kB, killing $pid" >&2
    kill -9 "$pid"
  fi
  sleep 1
done
wait "$pid"
rc=$?
echo "watchdog: exit $rc, peak RSS $((peak / 1000 / 1000)) GB" >&2
exit $rc
