# round-2 evidence: full GPU suite, bench lines of every workload, launch lists
mkdir -p gpurun_out/final
O=gpurun_out/final
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > $O/gputests.log 2>&1; echo tests_exit=$?; tail -1 $O/gputests.log
timeout 600 python bench.py > $O/bench_cfg5.json 2> $O/bench_cfg5.err; echo cfg5=$?
for w in cfg3 cfg2 cfg1; do timeout 300 python bench.py --workload $w --no-cpu-baseline > $O/bench_$w.json 2> $O/bench_$w.err; done
timeout 300 python bench.py --workload cfg4 --no-cpu-baseline > $O/bench_cfg4_fast.json 2> $O/bench_cfg4_fast.err
timeout 300 python bench.py --workload cfg4 --precision exact --no-cpu-baseline > $O/bench_cfg4_exact.json 2> $O/bench_cfg4_exact.err
timeout 300 python bench.py --precision fast-complex64 --no-cpu-baseline > $O/bench_cfg5_c64.json 2> $O/bench_cfg5_c64.err
timeout 600 python bench.py --impl reference > $O/bench_reference_arm.json 2> $O/bench_reference_arm.err
for f in $O/bench_*.json; do python -c "
import json,sys; d=json.load(open('$f')); r=d.get('roofline') or {}; e=d.get('e2e') or {}
print('$f'.split('/')[-1], round(d['value']/1e9,4), 'G', round(d['ms_per_step'],4), 'ms frac', round(r.get('frac',0) or 0,3), 'e2e', round((e.get('value') or 0)/1e9,3), 'clk', (d.get('clocks') or {}).get('sm_mhz'))" 2>/dev/null || echo "$f failed"; done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
ncu --metrics $M --clock-control none --csv --log-file $O/launch_cfg5.csv python scripts/profile_cycle.py --dim 3 --level 6 --k 80 --cycles 2 > /dev/null 2>&1
ncu --metrics $M --clock-control none --csv --log-file $O/launch_cfg4_fast.csv python scripts/amr_cycle.py 2 fast > /dev/null 2>&1
ls $O
