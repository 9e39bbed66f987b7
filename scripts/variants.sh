#!/bin/bash
# Developer A/B of compile-time variants: scripts/variants.sh "cfg5 cfg3" "base variants/x.so ..."
# base = the in-tree library.  Prints value / ms per cycle / fine-pass ms per run.
for w in $1; do for v in $2; do for rep in 1 2; do
  if [ "$v" = base ]; then lib=""; else lib="TMG_LIB=$PWD/$v"; fi
  env $lib python bench.py --workload $w --no-cpu-baseline --no-e2e --steps 20 > gpurun_out/var.json 2>gpurun_out/var.err
  python -c "
import json; d=json.load(open('gpurun_out/var.json')); print('$w $v', round(d['value']/1e9,2), round(d['ms_per_step'],4), round(d.get('fine_pass_ms',0),4), d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -3 gpurun_out/var.err
done; done; done
