#!/bin/bash
# round-2 session: full GPU suite, variant A/B, FP64 peak, complex64 bench
mkdir -p gpurun_out
./scripts/fp64_peak > gpurun_out/fp64_peak.json 2>&1
timeout 1500 python -m pytest tests -m gpu -q -s -x --timeout 900 > gpurun_out/gputests.log 2>&1
tail -25 gpurun_out/gputests.log
timeout 600 bash scripts/variants.sh "cfg5" "base variants/nosc.so" > gpurun_out/var.log 2>&1
cat gpurun_out/var.log
timeout 300 python bench.py --precision fast-complex64 --no-cpu-baseline > gpurun_out/bench_c64.json 2> gpurun_out/bench_c64.err
tail -c 1500 gpurun_out/bench_c64.json; tail -3 gpurun_out/bench_c64.err
cat gpurun_out/fp64_peak.json
