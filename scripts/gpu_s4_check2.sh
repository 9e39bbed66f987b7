# session 4: after the phase-B task map (fused3 r1 / r2): full GPU suite + bench lines of the 3D workloads
mkdir -p gpurun_out/s4b
O=gpurun_out/s4b
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider -x > $O/gputests.log 2>&1; echo tests_exit=$?; tail -1 $O/gputests.log
for w in cfg3 cfg5; do timeout 300 python bench.py --workload $w --no-cpu-baseline --no-e2e > $O/bench_$w.json 2> $O/bench_$w.err; done
timeout 300 python bench.py --precision fast-complex64 --no-cpu-baseline --no-e2e > $O/bench_cfg5_c64.json 2> $O/bench_cfg5_c64.err
timeout 300 python bench.py --workload cfg3 --precision fast-complex64 --no-cpu-baseline --no-e2e > $O/bench_cfg3_c64.json 2> $O/bench_cfg3_c64.err
for f in $O/bench_*.json; do python -c "
import json,sys; d=json.load(open('$f')); r=d.get('roofline') or {}
print('$f'.split('/')[-1], round(d['value']/1e9,4), 'G', round(d['ms_per_step'],4), 'ms fine', round(d.get('fine_pass_ms',0),4), 'clk', (d.get('clocks') or {}).get('sm_mhz'), (d.get('clocks') or {}).get('reasons'))" 2>/dev/null || echo "$f failed"; done
