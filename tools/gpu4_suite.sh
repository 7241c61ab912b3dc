# 4-GPU box: the whole GPU suite (virtual-rank meshes incl. a dense-model
# trainer spread over the 4 GPUs, multi-process NCCL meshes), then 4x1 / 2x2
# bench lines.  usage: bash tools/gpu4_suite.sh OUTDIR
set -u
O=${1:-gpurun_out/g4}
mkdir -p $O
python -m paper_2508_03854_b200.build > /dev/null 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest.log 2>&1
echo "pytest rc=$?"; tail -3 $O/pytest.log
run() {  # name nproc args...
  local name=$1 np=$2; shift 2
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $np --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) bench.py --gpus $np "$@" > $O/$name.json 2> $O/$name.err
  echo "$name rc=$?"; python -c "
import json; d=json.load(open('$O/$name.json')); print('$name', round(d.get('value'),0), round(d.get('ms_per_step'),4), (d.get('e2e') or {}).get('value'))" 2>/dev/null || tail -3 $O/$name.err
}
run n4 4 --steps 20 --warmup 5 --no-cpu-baseline
run 2x2 4 --steps 20 --warmup 5 --mesh 2x2 --no-cpu-baseline
