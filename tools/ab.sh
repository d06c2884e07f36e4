# A/B of env settings in one GPU session: bash tools/ab.sh "ENV_A" "ENV_B" [config] [rounds]
A="$1"; B="$2"; CFG="${3:-2}"; R="${4:-3}"
mkdir -p gpurun_out
for i in $(seq 1 $R); do
  for e in "$A" "$B"; do
    echo "[$e]" >> gpurun_out/ab.txt
    env $e python tools/level_profile.py $CFG tup strided >> gpurun_out/ab.txt 2>&1
  done
done
