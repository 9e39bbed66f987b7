#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/gputests.log 2>&1; tail -3 gpurun_out/gputests.log
for v in base variants/r1ty8.so; do
  if [ "$v" = base ]; then lib=""; else lib="TMG_LIB=$PWD/$v"; fi
  for rep in 1 2; do env $lib python bench.py --precision fast-complex64 --no-cpu-baseline --no-e2e > gpurun_out/v.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/v.json')); print('c64 $v', round(d['value']/1e9,2), round(d['ms_per_step'],4), round(d['fine_pass_ms'],4), d['clocks']['sm_mhz'], d['clocks']['reasons'])"; done
done
timeout 900 bash scripts/variants.sh "cfg5 cfg3 cfg2 cfg1" "base" > gpurun_out/var.log 2>&1; cat gpurun_out/var.log
