# cfg4 quick: AMR parity tests, bench, launch list of 2 cycles
mkdir -p gpurun_out
timeout 600 python -m pytest -q -m gpu -p no:cacheprovider tests/test_gpu_amr.py tests/test_gpu_goldens.py tests/test_gpu_dynamic.py > gpurun_out/gputests_amr.log 2>&1; echo tests_exit=$?
tail -2 gpurun_out/gputests_amr.log
timeout 300 python bench.py --workload cfg4 --no-cpu-baseline > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err; echo bench=$?
python -c "
import json; d=json.load(open('gpurun_out/bench_cfg4.json')); print('cfg4', round(d['value']/1e9,3), 'G', round(d['ms_per_step'],4), 'ms')"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launch_cfg4.csv python scripts/amr_cycle.py 2 > gpurun_out/ncu_cfg4.log 2>&1
python scripts/summarize_ncu.py launches gpurun_out/launch_cfg4.csv | tail -22
