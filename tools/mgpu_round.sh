# 4-GPU box: multi-process NCCL mesh parity at HEAD + mesh bench lines (cfg3 tables).
set -u
mkdir -p gpurun_out
python -m paper_2508_03854_b200.build > /dev/null 2>&1
nvidia-smi topo -m > gpurun_out/mg_topo.txt 2>&1
timeout 1500 python -m pytest tests/test_multigpu.py -q -k "test_mesh_parity[" --timeout 600 > gpurun_out/mg_pytest.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/mg_pytest.log
run() {  # name nproc args...
  local name=$1 np=$2; shift 2
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $np --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) bench.py --gpus $np "$@" > gpurun_out/mg_$name.json 2> gpurun_out/mg_$name.err
  echo "$name rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/mg_$name.json')); print('$name', d.get('value'), d.get('ms_per_step'), d.get('e2e',{}).get('value'))" 2>/dev/null
}
run n2 2 --steps 20 --warmup 5 --no-cpu-baseline
run n4 4 --steps 20 --warmup 5 --no-cpu-baseline
run 2x2 4 --steps 20 --warmup 5 --mesh 2x2 --no-cpu-baseline
run 1x4 4 --steps 20 --warmup 5 --mesh 1x4 --no-cpu-baseline
