# Round-2 evidence on ONE GPU (run under gpurun; read/summarise here with
# tools/ncu_summarize.py).  The N > 1 kernels run on a 2x2 mesh of virtual
# ranks (LocalHub) so they are captured on a single B200 as well.
set -u
mkdir -p gpurun_out
TAG=${TAG:-v3}
python -m paper_2508_03854_b200.build > /dev/null 2>&1
python bench.py --steps 50 --warmup 5 > gpurun_out/bench_${TAG}_n1.json 2> gpurun_out/bench_${TAG}_n1.err
echo "bench rc=$?"
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_${TAG}_reference_n1.json 2> gpurun_out/ref.err
echo "reference rc=$?"
python tools/gather_probe.py > gpurun_out/gather_probe_${TAG}.txt 2>&1
echo "gather probe rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
echo "launch list rc=$?"
for k in k_lookup_ring k_update_ring k_range_partials k_radix_pass k_radix_hist k_group_partials; do
  ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip 2 -c 1 \
      -o gpurun_out/full_$k -f python tools/step_driver.py --steps 3 > gpurun_out/ncu_$k.log 2>&1
  echo "$k rc=$?"
done
# N > 1 kernels: 2x2 mesh (cfg3 tables, table-wise) and 2x1 row-wise (multi-owner bags), B = 8192 per rank
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}_mesh2x2.csv \
    python tools/step_driver.py --config cfg3 --mesh 2x2 --batch 8192 --steps 2 > gpurun_out/ncu_mesh_launch.log 2>&1
echo "mesh launch list rc=$?"
for k in k_bucket_count k_bucket_permute k_combine k_grad_gather k_p2p_push k_p2p_mean k_p2p_scatter k_flag_count k_flag_write k_mark_slots k_publish_counts; do
  ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip 4 -c 1 \
      -o gpurun_out/full_$k -f python tools/step_driver.py --config cfg3 --mesh 2x2 --batch 8192 --steps 3 \
      > gpurun_out/ncu_$k.log 2>&1
  echo "$k rc=$?"
done
cuobjdump -sass paper_2508_03854_b200/libsparse2d_b200.so > gpurun_out/sass_all.txt 2>&1
echo done
