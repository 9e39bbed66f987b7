#!/bin/bash
# Developer A/B of runtime switches: scripts/envab.sh "cfg1 cfg2" "X=1 X=0" [reps]
# Prints value / ms per cycle / fine-pass ms per run.
reps=${3:-2}
for w in $1; do for r in $(seq $reps); do for v in $2; do
  env $v python bench.py --workload $w --no-cpu-baseline --no-e2e --steps 20 > gpurun_out/var.json 2>gpurun_out/var.err
  python -c "
import json; d=json.load(open('gpurun_out/var.json')); print('$w $v', round(d['value']/1e9,2), round(d['ms_per_step'],4), round(d.get('fine_pass_ms',0),4), d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -3 gpurun_out/var.err
done; done; done
