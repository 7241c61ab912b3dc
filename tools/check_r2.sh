# 1 GPU: dense-model trainer parity, core parity, bench.  usage: bash tools/check_r2.sh OUTDIR
set -u
O=${1:-gpurun_out/c2}
mkdir -p $O
python -m paper_2508_03854_b200.build > $O/build.log 2>&1 || { echo build failed; tail -20 $O/build.log; exit 1; }
timeout 600 python -m pytest tests/test_local_mesh.py -q -x -k dense > $O/pytest_dense.log 2>&1
echo "dense rc=$?"; tail -15 $O/pytest_dense.log
timeout 1200 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1
echo "pytest rc=$?"; tail -3 $O/pytest.log
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > $O/bench.json 2> $O/bench.err
python -c "
import json; d=json.load(open('$O/bench.json')); print(round(d['ms_per_step'],4), {k: round(v,4) for k,v in d['phase_split_ms'].items()})" || tail -5 $O/bench.err
