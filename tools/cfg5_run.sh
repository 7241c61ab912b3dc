# 4-GPU box: config 5 (500 tables, D 32-256, pooling 1-200, B = 32768 / GPU) on the 2x2 mesh,
# momentum-scaled (c = 4, the config's)  and plain row-wise AdaGrad (c = 1).  usage: bash tools/cfg5_run.sh OUTDIR
set -u
O=${1:-gpurun_out/cfg5}
mkdir -p $O
python -m paper_2508_03854_b200.build > /dev/null 2>&1
free -g | head -2
# B = 32768 / GPU does not fit on the 2x2 mesh: the replica sync's dirty-row
# staging (rows x (max dim + 4) x 4 B at D_max = 256) alone needs ~50 GB per
# GPU beside 38 GB of shards and ~60 GB of batch buffers (measured: OOM in
# the first sync, gpurun_out/cfg5b); the largest power of two that fits is
# 16384 (BATCH=... overrides)
BATCH=${BATCH:-16384}
echo "per-GPU batch $BATCH"
if [ "${PARITY:-1}" = 1 ]; then
  timeout 900 python -m pytest tests/test_multigpu.py -m gpu -q > $O/pytest.log 2>&1
  echo "pytest rc=$?"; tail -2 $O/pytest.log
fi
run() {  # name args...
  local name=$1; shift
  timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) bench.py --gpus 4 "$@" > $O/$name.json 2> $O/$name.err
  echo "$name rc=$?"; python -c "
import json; d=json.load(open('$O/$name.json')); print('$name', d['step_stats'], round(d.get('value'),0), round(d.get('ms_per_step'),3), d['config'].get('per_gpu_batch'), d.get('step_stats',{}).get('sync_mode'), {k: round(v,3) for k,v in d.get('phase_split_ms',{}).items()})" 2>/dev/null || tail -5 $O/$name.err
}
run cfg5_2x2_c4 --config cfg5 --mesh 2x2 --steps 5 --warmup 3 --nbatches 1 --batch $BATCH --c 4 --no-cpu-baseline --no-e2e
run cfg5_2x2_c1 --config cfg5 --mesh 2x2 --steps 5 --warmup 3 --nbatches 1 --batch $BATCH --c 1 --no-cpu-baseline --no-e2e
run cfg3_2x2 --mesh 2x2 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e
