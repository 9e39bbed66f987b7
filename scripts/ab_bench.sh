#!/bin/bash
# A/B of env settings over workloads: scripts/ab_bench.sh "cfg5 cfg3" "TMG_CHAIN=1 TMG_CHAIN=0"
for w in $1; do for e in $2; do
  env $e python bench.py --workload $w --no-cpu-baseline --steps 10 > gpurun_out/ab.json 2>gpurun_out/ab.err
  python -c "
import json; d=json.load(open('gpurun_out/ab.json')); print('$w $e', round(d['value']/1e9,2), round(d['ms_per_step'],4), round(d.get('fine_pass_ms',0),4), round(d['roofline']['frac'],3))" || tail -3 gpurun_out/ab.err
done; done
