python -m paper_2508_03854_b200.build >/dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full_size.py -q -x 2>&1 | tail -3
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_sort.csv python tools/step_driver.py --steps 3 > gpurun_out/ncu_sort.log 2>&1
python tools/launch_table.py gpurun_out/launches_sort.csv 22
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_sort.json 2> gpurun_out/bench_sort.err
python -c "
import json; d=json.load(open('gpurun_out/bench_sort.json')); print(d['ms_per_step'], d['phase_split_ms'])"
