# cfg4 in fast / exact precision: AMR tests, bench lines (fast fused / fast unfused / exact), fast launch list
mkdir -p gpurun_out
timeout 600 python -m pytest -q -m gpu -p no:cacheprovider tests/test_gpu_amr.py tests/test_gpu_amr_fast.py > gpurun_out/gputests_amr.log 2>&1; echo tests_exit=$?
tail -2 gpurun_out/gputests_amr.log
for v in "fast 1" "fast 0" "exact 1"; do set -- $v
TMG_AMR_FUSED=$2 timeout 300 python bench.py --workload cfg4 --precision $1 --no-cpu-baseline > gpurun_out/bench_cfg4_$1$2.json 2> gpurun_out/bench_cfg4_$1$2.err; echo bench=$?
python -c "
import json; d=json.load(open('gpurun_out/bench_cfg4_$1$2.json')); print('cfg4 $1 fused=$2', round(d['value']/1e9,3), 'G', round(d['ms_per_step'],4), 'ms e2e', round(d['e2e']['value']/1e9,3))"
done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launch_cfg4_fast.csv python scripts/amr_cycle.py 2 fast > gpurun_out/ncu_cfg4.log 2>&1
python scripts/summarize_ncu.py launches gpurun_out/launch_cfg4_fast.csv | tail -21
