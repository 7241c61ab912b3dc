#!/bin/bash
# One GPU: bench line (+ cpu baseline), reference arm, ncu launch list and
# `ncu --set full` captures of the three hot kernels.  Run under gpurun; then
# python tools/ncu_summarize.py --round <r> --tag <t> --full gpurun_out/full_*.ncu-rep \
#     --launches gpurun_out/launches.csv
set -u
mkdir -p gpurun_out
python bench.py --steps 50 --warmup 5 > gpurun_out/final_n1.json 2> gpurun_out/final_n1.err
echo "bench rc=$?"
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ref_n1.json 2> gpurun_out/ref_n1.err
echo "reference rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
echo "launch list rc=$?"
for k in k_update_ring k_lookup_ring k_radix_pass k_range_partials; do
  ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip 2 -c 1 \
      -o gpurun_out/full_$k -f python tools/step_driver.py --steps 3 > gpurun_out/ncu_$k.log 2>&1
  echo "$k rc=$?"
done
