#!/bin/bash
# launch lists (2 cycles) of the current build + one ncu --set full of the 2D fused pass
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
python scripts/profile_cycle.py --dim 2 --level 7 --k 100 --bpx --cycles 2 > gpurun_out/plain2.log 2>&1 && \
python scripts/profile_cycle.py --dim 3 --level 6 --k 80 --cycles 2 > gpurun_out/plain5.log 2>&1 && \
python scripts/profile_cycle.py --dim 3 --level 5 --k 20 --cycles 2 > gpurun_out/plain3.log 2>&1 && \
python scripts/profile_cycle.py --dim 2 --level 5 --k 10 --cycles 2 > gpurun_out/plain1.log 2>&1 && {
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launch_cfg2.csv python scripts/profile_cycle.py --dim 2 --level 7 --k 100 --bpx --cycles 2 > /dev/null 2>&1
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launch_cfg5.csv python scripts/profile_cycle.py --dim 3 --level 6 --k 80 --cycles 2 > /dev/null 2>&1
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launch_cfg3.csv python scripts/profile_cycle.py --dim 3 --level 5 --k 20 --cycles 2 > /dev/null 2>&1
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launch_cfg1.csv python scripts/profile_cycle.py --dim 2 --level 5 --k 10 --cycles 2 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_fused2 -s 1 -c 1 -o gpurun_out/f2_2187_r2 python scripts/profile_cycle.py --dim 2 --level 7 --k 100 --bpx --cycles 2 > gpurun_out/ncu_f2.log 2>&1
}
ls gpurun_out/
