# 4-GPU A/B of the replica-sync paths on the 2x2 / 1x4 meshes (config 3).
# usage: bash tools/sync_ab.sh OUTDIR
set -u
O=${1:-gpurun_out/sab}
mkdir -p $O
python -m paper_2508_03854_b200.build > /dev/null 2>&1
timeout 600 python -m pytest tests/test_multigpu.py -q -x -k "local" 2>&1 | tail -2
run() {  # name env mesh
  local name=$1 envs=$2 mesh=$3
  env $envs timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) bench.py --gpus 4 --mesh $mesh --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > $O/$name.json 2> $O/$name.err
  python -c "
import json; d=json.load(open('$O/$name.json')); print('$name', round(d['ms_per_step'],4), d['step_stats']['sync_mode'], [round(r['ms'],1) for r in d['per_rank']], [max(r['step_ms']) for r in d['per_rank']], {k: round(v,3) for k,v in d['phase_split_ms'].items() if k.startswith('sync') or k=='update'})" 2>/dev/null || tail -3 $O/$name.err
}
run 2x2_snap "S2D_SYNC_SNAPSHOT=1" 2x2

run 2x2_slice "S2D_SYNC_SNAPSHOT=0" 2x2


run 1x4_slice "S2D_SYNC_SNAPSHOT=0" 1x4
