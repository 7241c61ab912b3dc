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
for k in k_bucket_count k_bucket_permute k_combine k_grad_gather k_pair_push k_pair_recv k_flag_count k_flag_write k_publish_counts; do
  ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip 4 -c 1 \
      -o gpurun_out/full_$k -f python tools/step_driver.py --config cfg3 --mesh 2x2 --batch 8192 --steps 3 \
      > gpurun_out/ncu_$k.log 2>&1
  echo "$k rc=$?"
done
# the M > 2 slice sync's kernels (forced on the 2x2 mesh)
for k in k_p2p_push k_p2p_mean k_p2p_scatter k_mark_slots; do
  S2D_SYNC_SNAPSHOT=0 ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip 4 -c 1 \
      -o gpurun_out/full_$k -f python tools/step_driver.py --config cfg3 --mesh 2x2 --batch 8192 --steps 3 \
      > gpurun_out/ncu_$k.log 2>&1
  echo "$k rc=$?"
done
# summarise on the box (the .ncu-rep files exceed what gpurun brings back)
OUT=gpurun_out/profile_out; mkdir -p $OUT
python tools/ncu_summarize.py --round r02 --tag ${TAG} --full gpurun_out/full_k_lookup_ring.ncu-rep \
    gpurun_out/full_k_update_ring.ncu-rep gpurun_out/full_k_range_partials.ncu-rep gpurun_out/full_k_radix_pass.ncu-rep \
    gpurun_out/full_k_radix_hist.ncu-rep gpurun_out/full_k_group_partials.ncu-rep --launches gpurun_out/launches_${TAG}.csv
cp profiles/r02/ncu_full_${TAG}_summary.csv $OUT/; cp profiles/r02/launches_${TAG}_summary.csv $OUT/
python tools/ncu_summarize.py --round r02 --tag ${TAG}_mesh2x2 --full gpurun_out/full_k_bucket_count.ncu-rep \
    gpurun_out/full_k_bucket_permute.ncu-rep gpurun_out/full_k_combine.ncu-rep gpurun_out/full_k_grad_gather.ncu-rep \
    gpurun_out/full_k_pair_push.ncu-rep gpurun_out/full_k_pair_recv.ncu-rep \
    gpurun_out/full_k_p2p_push.ncu-rep gpurun_out/full_k_p2p_mean.ncu-rep gpurun_out/full_k_p2p_scatter.ncu-rep \
    gpurun_out/full_k_flag_count.ncu-rep gpurun_out/full_k_flag_write.ncu-rep gpurun_out/full_k_mark_slots.ncu-rep \
    gpurun_out/full_k_publish_counts.ncu-rep --launches gpurun_out/launches_${TAG}_mesh2x2.csv
cp profiles/r02/ncu_full_${TAG}_mesh2x2_summary.csv $OUT/; cp profiles/r02/launches_${TAG}_mesh2x2_summary.csv $OUT/
cp profiles/traffic.json $OUT/
for k in k_lookup_ring k_update_ring k_range_partials k_radix_pass; do
  python tools/ncu_hot_src.py gpurun_out/full_$k.ncu-rep 30 > $OUT/hot_src_${TAG}_$k.txt 2>&1
done
cuobjdump -sass paper_2508_03854_b200/libsparse2d_b200.so 2>/dev/null | grep -E "Function :|UBLKCP|LDGSTS|F2F.F64.F32|SYNCS" \
    | awk '/Function :/{f=$0} !/Function :/{c[f" "$2]++} END{for (k in c) print c[k], k}' | sort -k2 > $OUT/sass_opcounts.txt
cp gpurun_out/bench_${TAG}_n1.json gpurun_out/bench_${TAG}_reference_n1.json gpurun_out/gather_probe_${TAG}.txt $OUT/
rm -f gpurun_out/*.ncu-rep gpurun_out/launches_*.csv
echo done
