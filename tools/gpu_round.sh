# One GPU pass for the round's evidence (run under gpurun from the repo root):
# tests, smoke, the default bench line, the ncu launch list of the bench command
# and one `ncu --set full` capture of the solve's top kernels (exported to csv).
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench.csv python bench.py --no-cpu-baseline --no-variants > gpurun_out/ncu_bench.log 2>&1; echo "ncu list rc=$?"
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"bsr3|dinv|csr_warp|csr_slice_strided|csr_pipe|cgs" -s 40 -c 16 -o gpurun_out/full_cfg2 -f python tools/profile_solve.py 2 tup 30 cgs > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
ncu -i gpurun_out/full_cfg2.ncu-rep --page raw --csv > gpurun_out/full_cfg2_raw.csv 2>/dev/null; echo "export rc=$?"
