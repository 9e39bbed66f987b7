#!/bin/bash
# final kernel: ncu --set full of k_fused3 at 729^3 (one launch)
mkdir -p gpurun_out
CMD="python bench.py --no-cpu-baseline --no-e2e --steps 2 --warmup 3"
$CMD > gpurun_out/plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:k_fused3 -s 3 -c 1 -o gpurun_out/f3_729_r2c $CMD > gpurun_out/ncu_f3.log 2>&1
tail -2 gpurun_out/ncu_f3.log
