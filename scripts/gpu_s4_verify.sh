# session-4 re-entry check: full GPU suite + the two target workloads
mkdir -p gpurun_out/s4
O=gpurun_out/s4
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > $O/gputests.log 2>&1; echo tests_exit=$?; tail -1 $O/gputests.log
timeout 600 python bench.py > $O/bench_cfg5.json 2> $O/bench_cfg5.err; echo cfg5=$?
timeout 300 python bench.py --workload cfg3 --no-cpu-baseline > $O/bench_cfg3.json 2> $O/bench_cfg3.err
for f in $O/bench_*.json; do python -c "
import json,sys; d=json.load(open('$f')); r=d.get('roofline') or {}; e=d.get('e2e') or {}
print('$f'.split('/')[-1], round(d['value']/1e9,4), 'G', round(d['ms_per_step'],4), 'ms frac', round(r.get('frac',0) or 0,3), 'e2e', round((e.get('value') or 0)/1e9,3), 'clk', (d.get('clocks') or {}).get('sm_mhz'), 'fine', d.get('fine_pass_ms'))" 2>/dev/null || echo "$f failed"; done
