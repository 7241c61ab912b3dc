# usage: bash tools/try_variants.sh "<sed expr per variant>"... ; runs parity + bench for each
set -u
f=${VARIANT_FILE:-paper_2508_03854_b200/csrc/k_stream.cu}
cp $f /tmp/orig.cu
i=0
for expr in "$@"; do
  cp /tmp/orig.cu $f
  sed -i "$expr" $f
  python -m paper_2508_03854_b200.build >/dev/null 2>&1 || { echo "build failed: $expr"; continue; }
  if [ $i -eq 0 ]; then timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full_size.py -q -x 2>&1 | tail -2; fi
  python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_var$i.json 2> gpurun_out/bench_var$i.err
  python -c "
import json; d=json.load(open('gpurun_out/bench_var$i.json')); print('$expr', round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['phase_split_ms'].items()})"
  i=$((i+1))
done
cp /tmp/orig.cu $f
