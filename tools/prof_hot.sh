# one GPU: full ncu captures of the hot N=1 kernels (cfg2) for reading here
set -u
mkdir -p gpurun_out
python -m paper_2508_03854_b200.build > /dev/null 2>&1
for k in k_lookup_ring k_update_ring k_range_partials; do
  ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip 2 -c 1 \
      -o gpurun_out/full_$k -f python tools/step_driver.py --steps 3 > gpurun_out/ncu_$k.log 2>&1
  echo "$k rc=$?"
done
