#!/bin/bash
# ncu evidence at the smaller BASELINE configs (run under gpurun from the repo root; outputs in gpurun_out/):
# per config a launch list of two GMRES iterations and one `ncu --set full` capture of one iteration's kernels.
mkdir -p gpurun_out
K='regex:bsr3|sell|bp3|srt_|csr_|dinv|panel_solve|band_solve|cgs|mgs|jtp|hsolve|coarse|presmooth|axpy'
for c in "$@"; do
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --profile-from-start off -k "$K" -c 200 --csv --log-file gpurun_out/ncu_launches_solve_cfg$c.csv \
    python tools/profile_solve.py $c tup 2 cgs strided > gpurun_out/ncu_launches_cfg$c.log 2>&1
  echo "launch list $c rc=$?"
  timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -k "$K" -c 60 \
    -o gpurun_out/full_cfg$c -f python tools/profile_solve.py $c tup 1 cgs strided > gpurun_out/ncu_full_cfg$c.log 2>&1
  echo "full capture $c rc=$?"
  ncu -i gpurun_out/full_cfg$c.ncu-rep --page raw --csv > gpurun_out/full_cfg${c}_raw.csv 2>/dev/null
  python tools/ncu_full_summary.py gpurun_out/full_cfg${c}_raw.csv gpurun_out/ncu_full_cfg$c.json \
    "ncu --set full --clock-control none, one GMRES(50) iteration of config $c (tools/profile_solve.py $c tup 1 cgs strided)"
  rm -f gpurun_out/full_cfg$c.ncu-rep gpurun_out/full_cfg${c}_raw.csv
done
du -sh gpurun_out
