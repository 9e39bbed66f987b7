# full GPU suite + bench lines (default workload, cfg3, cfg2)
timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/gputests.log 2>&1; echo tests_exit=$?
tail -3 gpurun_out/gputests.log
timeout 600 python bench.py > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err; echo bench_exit=$?
for w in cfg3 cfg2 cfg1 cfg4; do timeout 600 python bench.py --workload $w --no-cpu-baseline > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; done
for w in cfg5 cfg3 cfg2 cfg1 cfg4; do python -c "
import json; d=json.load(open('gpurun_out/bench_$w.json')); print('$w', round(d['value']/1e9,2), 'G', round(d['ms_per_step'],4), 'ms', 'frac', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value']/1e9,2), 'launches', d['gpu_launches'])"; done
