# A/B of environment settings: parity once (with the first setting), then a
# bench line per setting.  usage: bash tools/ab_envs.sh "A=1 B=2" "A=0" ...
set -u
python -m paper_2508_03854_b200.build > /dev/null 2>&1 || { echo build failed; exit 1; }
first=1
i=0
for s in "$@"; do
  if [ $first -eq 1 ]; then
    env $s timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full_size.py -q -x 2>&1 | tail -2
    first=0
  fi
  env $s python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/abe_$i.json 2> gpurun_out/abe_$i.err
  python -c "
import json; d=json.load(open('gpurun_out/abe_$i.json')); print('[$s]', round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['phase_split_ms'].items()})" || tail -3 gpurun_out/abe_$i.err
  i=$((i+1))
done
