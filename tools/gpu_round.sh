timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1])
print({k: d[k] for k in ('value','ms_per_step','e2e','gpu_launches','timing','variants')})
print(d['roofline']['achieved'], d['roofline']['frac'], d['precond_apply'], d['cpu_baseline']['value'], d['clocks'])"
