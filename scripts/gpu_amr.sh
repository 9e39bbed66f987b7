# cfg4: AMR parity tests, bench A/B (fused finest level vs separate), launch list
mkdir -p gpurun_out
timeout 900 python -m pytest -q -m gpu -p no:cacheprovider tests/test_gpu_amr.py tests/test_gpu_goldens.py tests/test_gpu_dynamic.py > gpurun_out/gputests_amr.log 2>&1; echo tests_exit=$?
tail -5 gpurun_out/gputests_amr.log
timeout 300 python bench.py --workload cfg4 --no-cpu-baseline > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err; echo bench=$?
TMG_AMR_FUSED=0 timeout 300 python bench.py --workload cfg4 --no-cpu-baseline > gpurun_out/bench_cfg4_unfused.json 2>> gpurun_out/bench_cfg4.err
for f in bench_cfg4 bench_cfg4_unfused; do python -c "
import json; d=json.load(open('gpurun_out/$f.json')); print('$f', round(d['value']/1e9,3), 'G', round(d['ms_per_step'],4), 'ms')"; done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launch_cfg4.csv python scripts/amr_cycle.py 2 > gpurun_out/ncu_cfg4.log 2>&1
python scripts/summarize_ncu.py launches gpurun_out/launch_cfg4.csv | tail -40
