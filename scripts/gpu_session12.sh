#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/gputests.log 2>&1; tail -3 gpurun_out/gputests.log
timeout 900 bash scripts/variants.sh "cfg5 cfg3" "base variants/prebtma.so" > gpurun_out/var.log 2>&1; cat gpurun_out/var.log
