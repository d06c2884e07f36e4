#!/bin/bash
# Round-2 evidence on one B200 (run under gpurun from the repo root; outputs in gpurun_out/):
#  1. the ncu launch list of the bench command (solve kernels only: the device setup's kernels are
#     filtered out by name), per-launch time and DRAM bytes, cold and serialized;
#  2. one `ncu --set full` capture of the solve's top kernels at config 5 (one GMRES iteration inside a
#     profiler range), exported to csv for tools/ncu_full_summary.py;
#  3. compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize.py.
mkdir -p gpurun_out
SOLVE='regex:bsr3|sell|bp3|srt_|csr_|dinv|panel_solve|band_solve|cgs|mgs|jtp|hsolve|coarse|presmooth|axpy|basis|backsub|start_cycle|norm|add_inplace|mcgs|cheb'
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k "$SOLVE" -c 400 --csv --log-file gpurun_out/ncu_launches_bench_cfg5.csv \
  python bench.py --steps 1 --warmup 1 --no-variants --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1
echo "launch list rc=$?"
timeout 1500 ncu --set full --import-source on --clock-control none --profile-from-start off \
  -k 'regex:bsr3|panel_solve|cgs|srt_|csr_warp|csr_slice|bp3|sell|jtp|dinv|hsolve' -c 44 \
  -o gpurun_out/full_cfg5 -f python tools/profile_solve.py 5 tup 1 cgs strided > gpurun_out/ncu_full.log 2>&1
echo "full capture rc=$?"
ncu -i gpurun_out/full_cfg5.ncu-rep --page raw --csv > gpurun_out/full_cfg5_raw.csv 2>/dev/null
python tools/ncu_full_summary.py gpurun_out/full_cfg5_raw.csv gpurun_out/ncu_full_cfg5.json \
  "ncu --set full --clock-control none, one GMRES(50) iteration of config 5 (tools/profile_solve.py 5 tup 1 cgs strided)"
# gpurun copies back at most 64 MiB: keep the report only when it is small
[ "$(stat -c %s gpurun_out/full_cfg5.ncu-rep 2>/dev/null || echo 0)" -gt 30000000 ] && rm -f gpurun_out/full_cfg5.ncu-rep
du -sh gpurun_out
if [ "$SKIP_SANITIZERS" != "1" ]; then for tool in memcheck racecheck synccheck; do
  timeout 1000 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize.py \
    > gpurun_out/sanitizer_$tool.log 2>&1
  echo "sanitizer $tool rc=$?"
done; fi
