# fast-cycle CUDA graphs: GPU suite, then A/B against TMG_GRAPH=0 on every workload
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider -x > gpurun_out/gputests.log 2>&1; echo tests_exit=$?
tail -3 gpurun_out/gputests.log
for w in cfg1 cfg2 cfg3 cfg5; do for g in 1 0; do
  TMG_GRAPH=$g timeout 300 python bench.py --workload $w --no-cpu-baseline --no-e2e > gpurun_out/g.json 2>gpurun_out/g.err
  python -c "
import json; d=json.load(open('gpurun_out/g.json')); print('$w graph=$g', round(d['value']/1e9,2), 'G', round(d['ms_per_step']*1e3,2), 'us', round(d.get('fine_pass_ms',0)*1e3,2), d['clocks']['sm_mhz'])" || tail -3 gpurun_out/g.err
done; done
