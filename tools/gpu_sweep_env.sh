# A/B sweep of one tuning env var over the C2 decode step: bash tools/gpu_sweep_env.sh VAR v1 v2 ...
var=$1; shift
for v in "$@"; do
  env $var=$v timeout 300 python bench.py --no-extras --no-cpu-baseline --steps 128 2>/dev/null | tail -1 > gpurun_out/sweep_$v.json
  python -c "import json; d=json.load(open('gpurun_out/sweep_$v.json')); print('$var=$v', round(d['value'],1), 'tok/s', round(d['ms_per_step'],4), 'ms')"
done
