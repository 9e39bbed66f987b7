#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/gputests.log 2>&1; tail -3 gpurun_out/gputests.log
python bench.py > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err; tail -c 300 gpurun_out/bench_cfg5.json
for w in cfg3 cfg2 cfg1; do python bench.py --workload $w --no-cpu-baseline > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err; done
python bench.py --precision fast-complex64 --no-cpu-baseline > gpurun_out/bench_cfg5_c64.json 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; cat gpurun_out/bench_ref.json | head -c 1500
CMD="python bench.py --no-cpu-baseline --no-e2e --steps 2 --warmup 3"
$CMD > gpurun_out/plain.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:k_fused3 -s 3 -c 1 -o gpurun_out/f3_729_r2b $CMD > gpurun_out/ncu_f3.log 2>&1
tail -2 gpurun_out/ncu_f3.log
