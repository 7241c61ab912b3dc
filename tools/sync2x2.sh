# 4-GPU box: pair-sync parity (virtual + NCCL meshes) and 2x2 bench lines.  usage: bash tools/sync2x2.sh OUTDIR
set -u
O=${1:-gpurun_out/s22}
mkdir -p $O
python -m paper_2508_03854_b200.build > /dev/null 2>&1
timeout 900 python -m pytest tests/test_multigpu.py tests/test_local_mesh.py -m gpu -q -x > $O/pytest.log 2>&1
echo "pytest rc=$?"; tail -2 $O/pytest.log
for i in 1 2; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) bench.py --gpus 4 --mesh 2x2 --steps 30 --warmup 5 --no-cpu-baseline --no-e2e > $O/2x2_$i.json 2> $O/2x2_$i.err
  python -c "
import json; d=json.load(open('$O/2x2_$i.json')); print('2x2', round(d['value']/1e6,2), round(d['ms_per_step'],4), {k: round(v,3) for k,v in d['phase_split_ms'].items() if k.startswith('sync') or k in ('update','lookup')})" || tail -3 $O/2x2_$i.err
done
