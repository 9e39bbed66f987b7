# session-4 closing run: full GPU suite, smoke, bench lines of every workload + the reference arm
mkdir -p gpurun_out/s4h
O=gpurun_out/s4h
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > $O/gputests.log 2>&1; echo tests_exit=$?; tail -1 $O/gputests.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?; tail -1 $O/smoke.log
timeout 600 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > $O/bench_reference_arm.json 2> $O/bench_reference_arm.err; echo ref=$?
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench_cfg5.json 2> $O/bench_cfg5.err; echo cfg5=$?
for w in cfg3 cfg2 cfg1; do timeout 300 python bench.py --workload $w --no-cpu-baseline > $O/bench_$w.json 2> $O/bench_$w.err; done
timeout 300 python bench.py --workload cfg4 --no-cpu-baseline > $O/bench_cfg4_fast.json 2> $O/bench_cfg4_fast.err
timeout 300 python bench.py --workload cfg4 --precision exact --no-cpu-baseline > $O/bench_cfg4_exact.json 2> $O/bench_cfg4_exact.err
timeout 300 python bench.py --precision fast-complex64 --no-cpu-baseline > $O/bench_cfg5_c64.json 2> $O/bench_cfg5_c64.err
timeout 300 python bench.py --workload cfg2 --precision fast-complex64 --no-cpu-baseline > $O/bench_cfg2_c64.json 2> $O/bench_cfg2_c64.err
for f in $O/bench_*.json; do python -c "
import json,sys; d=json.load(open('$f')); r=d.get('roofline') or {}; e=d.get('e2e') or {}
print('$f'.split('/')[-1], round(d['value']/1e9,4), 'G', round(d['ms_per_step'],4), 'ms frac', round(r.get('frac',0) or 0,3), 'e2e', round((e.get('value') or 0)/1e9,3), 'clk', (d.get('clocks') or {}).get('sm_mhz'), 'fine', d.get('fine_pass_ms'))" 2>/dev/null || echo "$f failed"; done
timeout 300 python bench.py --steps 400 --warmup 5 --no-cpu-baseline --no-e2e > $O/sustained400.json 2> $O/sustained400.err
python -c "
import json; d=json.load(open('$O/sustained400.json')); print('sustained400', round(d['value']/1e9,2), d['ms_per_step'], d['clocks'])"
CMD="python bench.py --no-cpu-baseline --no-e2e --steps 2 --warmup 3"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_bench_cfg5.csv $CMD > $O/ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_fused3 -s 3 -c 1 -o $O/f3_729 $CMD > $O/ncu_f3.log 2>&1
python scripts/summarize_ncu.py full $O/f3_729.ncu-rep | head -8
