# 4-GPU box: N = 1, 2, 4 (N x 1, config 3 tables) and the 2x2 mesh at HEAD.  usage: bash tools/scale4.sh OUTDIR
set -u
O=${1:-gpurun_out/sc4}
mkdir -p $O
python -m paper_2508_03854_b200.build > /dev/null 2>&1
for np in 1 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $np --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) bench.py --gpus $np --steps 20 --warmup 5 --no-cpu-baseline > $O/n$np.json 2> $O/n$np.err
  python -c "
import json; d=json.load(open('$O/n$np.json')); print('n$np', round(d['value']/1e6,2), round(d['ms_per_step'],4), round(d['e2e']['value']/1e6,2))" || tail -3 $O/n$np.err
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) bench.py --gpus 4 --mesh 2x2 --steps 20 --warmup 5 --no-cpu-baseline > $O/2x2.json 2> $O/2x2.err
python -c "
import json; d=json.load(open('$O/2x2.json')); print('2x2', round(d['value']/1e6,2), round(d['ms_per_step'],4), round(d['e2e']['value']/1e6,2))" || tail -3 $O/2x2.err
