# 4-GPU box: config 4 (4 x 200M x 128 bf16 row-wise, fp32 moments) on the 2x2 mesh, raw Zipf
# (rank = row, as the reference generator) and scrambled ids.  usage: bash tools/cfg4_run.sh OUTDIR
set -u
O=${1:-gpurun_out/cfg4}
mkdir -p $O
python -m paper_2508_03854_b200.build > /dev/null 2>&1
run() {  # name args...
  local name=$1; shift
  timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) bench.py --gpus 4 "$@" > $O/$name.json 2> $O/$name.err
  echo "$name rc=$?"; python -c "
import json; d=json.load(open('$O/$name.json')); print('$name', d['step_stats'], round(d.get('value'),0), round(d.get('ms_per_step'),3), {k: round(v,3) for k,v in d.get('phase_split_ms',{}).items()})" 2>/dev/null || tail -5 $O/$name.err
}
run cfg4_2x2_raw --config cfg4 --mesh 2x2 --steps 10 --warmup 3 --nbatches 1 --no-cpu-baseline --no-e2e
run cfg4_2x2_scrambled --config cfg4 --mesh 2x2 --steps 10 --warmup 3 --nbatches 1 --scramble --no-cpu-baseline --no-e2e
