#!/bin/bash
# variants A/B of the fused pass, then one ncu --set full capture of k_fused3 at 729^3
mkdir -p gpurun_out
timeout 900 bash scripts/variants.sh "cfg5 cfg3" "base variants/nosc.so variants/minb2.so" > gpurun_out/var.log 2>&1
cat gpurun_out/var.log
CMD="python bench.py --no-cpu-baseline --no-e2e --steps 2 --warmup 3"
$CMD > gpurun_out/plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:k_fused3 -s 3 -c 1 -o gpurun_out/f3_729_r2a $CMD > gpurun_out/ncu_f3.log 2>&1
tail -3 gpurun_out/ncu_f3.log
