mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_bench.csv python bench.py --no-cpu-baseline --no-variants > gpurun_out/ncu_bench.log 2>&1; echo "ncu list rc=$?"
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"bsr3|dinv|csr_pipe|mgs_fast" -s 40 -c 14 -o gpurun_out/full_cfg2 -f python tools/profile_solve.py 2 tup 30 > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
