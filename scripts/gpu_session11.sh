#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/gputests.log 2>&1; tail -3 gpurun_out/gputests.log
timeout 900 bash scripts/variants.sh "cfg5 cfg3" "base variants/prebtma.so" > gpurun_out/var.log 2>&1; cat gpurun_out/var.log
for rep in 1 2; do python bench.py --precision fast-complex64 --no-cpu-baseline --no-e2e > gpurun_out/v.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/v.json')); print('c64 base', round(d['value']/1e9,2), round(d['ms_per_step'],4), round(d['fine_pass_ms'],4), d['clocks']['sm_mhz'], d['clocks']['reasons'])"; done
