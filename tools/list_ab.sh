# 4-GPU box: NCCL mesh parity, then the dirty-list sync A/B on cfg4 / cfg3 2x2.  usage: bash tools/list_ab.sh OUTDIR
set -u
O=${1:-gpurun_out/lab}
mkdir -p $O
python -m paper_2508_03854_b200.build > /dev/null 2>&1
timeout 900 python -m pytest tests/test_multigpu.py -m gpu -q > $O/pytest.log 2>&1
echo "pytest rc=$?"; tail -2 $O/pytest.log
run() {  # name env args...
  local name=$1 envs=$2; shift 2
  env $envs timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) bench.py --gpus 4 "$@" > $O/$name.json 2> $O/$name.err
  python -c "
import json; d=json.load(open('$O/$name.json')); print('$name', round(d.get('value')/1e6,2), round(d.get('ms_per_step'),3), {k: round(v,3) for k,v in d.get('phase_split_ms',{}).items() if k.startswith('sync') or k == 'update'})" 2>/dev/null || tail -5 $O/$name.err
}
run cfg4_raw_list "" --config cfg4 --mesh 2x2 --steps 10 --warmup 3 --nbatches 1 --no-cpu-baseline --no-e2e
run cfg4_raw_flags "S2D_SYNC_LIST=0" --config cfg4 --mesh 2x2 --steps 10 --warmup 3 --nbatches 1 --no-cpu-baseline --no-e2e
run cfg4_scr_list "" --config cfg4 --mesh 2x2 --steps 10 --warmup 3 --nbatches 1 --scramble --no-cpu-baseline --no-e2e
run cfg3_2x2_list "" --mesh 2x2 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e
run cfg3_2x2_flags "S2D_SYNC_LIST=0" --mesh 2x2 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e
