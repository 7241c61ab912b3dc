# A/B of an environment switch: parity once, then bench with VAR=each value.
# usage: bash tools/ab_env.sh VAR v1 v2 ...
set -u
var=$1; shift
python -m paper_2508_03854_b200.build > /dev/null 2>&1 || { echo build failed; exit 1; }
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full_size.py tests/test_gpu_full_config.py -q -x -k "not cfg4 and not cfg5" 2>&1 | tail -2
for v in "$@"; do
  env $var=$v python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/ab_$v.json 2> gpurun_out/ab_$v.err
  python -c "
import json; d=json.load(open('gpurun_out/ab_$v.json')); print('$var=$v', round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['phase_split_ms'].items()})"
done
