# 4-GPU box: NCCL mesh parity + 2D mesh bench lines, cfg4 / cfg5 at spec.
# usage: bash tools/mgpu_round3.sh OUTDIR [skip-pytest]
set -u
O=${1:-gpurun_out/mg3}
mkdir -p $O
python -m paper_2508_03854_b200.build > /dev/null 2>&1
if [ "${2:-}" != "skip-pytest" ]; then
  timeout 900 python -m pytest tests/test_multigpu.py tests/test_local_mesh.py -q -x -k "local or replica or sync or trainer or mesh_matches" > $O/pytest_local.log 2>&1
  echo "pytest local rc=$?"; tail -2 $O/pytest_local.log
  timeout 1500 python -m pytest tests/test_multigpu.py -q -k "test_mesh_parity[" --timeout 600 > $O/pytest.log 2>&1
  echo "pytest rc=$?"; tail -3 $O/pytest.log
fi
run() {  # name nproc args...
  local name=$1 np=$2; shift 2
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $np --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) bench.py --gpus $np "$@" > $O/$name.json 2> $O/$name.err
  echo "$name rc=$?"; python -c "
import json; d=json.load(open('$O/$name.json')); print('$name', round(d.get('value'),0), round(d.get('ms_per_step'),4), (d.get('e2e') or {}).get('value'), d.get('step_stats',{}).get('sync_mode'), {k: round(v,3) for k,v in d.get('phase_split_ms',{}).items()})" 2>/dev/null || tail -3 $O/$name.err
}
run n1 1 --steps 20 --warmup 5 --no-cpu-baseline
run 2x2 4 --steps 20 --warmup 5 --mesh 2x2 --no-cpu-baseline
run 1x4 4 --steps 20 --warmup 5 --mesh 1x4 --no-cpu-baseline
run n4 4 --steps 20 --warmup 5 --no-cpu-baseline
run n2 2 --steps 20 --warmup 5 --no-cpu-baseline
run cfg4_2x2_raw 4 --config cfg4 --mesh 2x2 --steps 10 --warmup 3 --nbatches 1 --no-cpu-baseline --no-e2e
run cfg4_2x2_scrambled 4 --config cfg4 --mesh 2x2 --steps 10 --warmup 3 --nbatches 1 --scramble --no-cpu-baseline --no-e2e
run cfg5_2x2_cM 4 --config cfg5 --mesh 2x2 --steps 5 --warmup 3 --nbatches 1 --batch 16384 --no-cpu-baseline --no-e2e
run cfg5_2x2_c1 4 --config cfg5 --mesh 2x2 --steps 5 --warmup 3 --nbatches 1 --batch 16384 --c 1 --no-cpu-baseline --no-e2e
