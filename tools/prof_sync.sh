# ncu captures of the snapshot replica-sync kernels on a 2x2 mesh of virtual
# ranks on one GPU (config 3 tables, B = 16384 per rank); summaries only.
set -u
OUT=gpurun_out/prof_sync; mkdir -p $OUT
python -m paper_2508_03854_b200.build > /dev/null 2>&1
for k in k_sg_mean k_sg_push k_update_ring; do
  tag=$(echo "$k" | tr -c 'a-z0-9_\n' '_')
  ncu --set full --clock-control none --import-source on -k "regex:${k%%<*}" --launch-skip 4 -c 2 \
      -o gpurun_out/full_$tag -f python tools/step_driver.py --config cfg3 --mesh 2x2 --batch 16384 --steps 4 \
      > $OUT/ncu_$tag.log 2>&1
  echo "$k rc=$?"
  ncu -i gpurun_out/full_$tag.ncu-rep --page details --csv > $OUT/details_$tag.csv 2>&1
  python tools/ncu_hot_src.py gpurun_out/full_$tag.ncu-rep 30 > $OUT/hot_src_$tag.txt 2>&1
done
rm -f gpurun_out/*.ncu-rep
echo done
