# A/B of env settings on the bench value in one GPU session: bash tools/ab_bench.sh rounds "ENV_A" "ENV_B" ...
R="$1"; shift
mkdir -p gpurun_out
for i in $(seq 1 $R); do
  for e in "$@"; do
    v=$(env $e python bench.py --no-cpu-baseline --no-variants --steps 3 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['avg_launch_ms'], d['precond_apply']['ms'])")
    echo "[$e] $v" >> gpurun_out/ab_bench.txt
  done
done
