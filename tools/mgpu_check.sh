# 4-GPU box: multi-process NCCL mesh parity at HEAD + mesh bench lines (config 3 tables).
# usage: bash tools/mgpu_check.sh OUTDIR
set -u
O=${1:-gpurun_out/mgc}
mkdir -p $O
python -m paper_2508_03854_b200.build > /dev/null 2>&1
timeout 900 python -m pytest tests/test_multigpu.py -m gpu -q -x > $O/pytest.log 2>&1
echo "pytest rc=$?"; tail -2 $O/pytest.log
run() {  # name env nproc args...
  local name=$1 envs=$2 np=$3; shift 3
  env $envs timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $np --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) bench.py --gpus $np "$@" > $O/$name.json 2> $O/$name.err
  echo "$name rc=$?"; python -c "
import json; d=json.load(open('$O/$name.json')); print('$name', round(d.get('value'),0), round(d.get('ms_per_step'),4), (d.get('e2e') or {}).get('value'), d.get('step_stats',{}).get('sync_mode'), {k: round(v,3) for k,v in d.get('phase_split_ms',{}).items()})" 2>/dev/null || tail -3 $O/$name.err
}
run n4 "" 4 --steps 20 --warmup 5 --no-cpu-baseline
run 2x2 "" 4 --steps 20 --warmup 5 --mesh 2x2 --no-cpu-baseline
run 2x2_slice "S2D_SYNC_SNAPSHOT=0" 4 --steps 20 --warmup 5 --mesh 2x2 --no-cpu-baseline --no-e2e
run 1x4 "" 4 --steps 20 --warmup 5 --mesh 1x4 --no-cpu-baseline --no-e2e
run n2 "" 2 --steps 20 --warmup 5 --no-cpu-baseline
