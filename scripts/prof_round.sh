# launch lists (2 cycles) of the current build for cfg2 / cfg3 / cfg5 / cfg1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launch_cfg2.csv python scripts/profile_cycle.py --dim 2 --level 7 --k 100 --bpx --cycles 2 > /dev/null 2>&1
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launch_cfg3.csv python scripts/profile_cycle.py --dim 3 --level 5 --k 20 --cycles 2 > /dev/null 2>&1
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launch_cfg5.csv python scripts/profile_cycle.py --dim 3 --level 6 --k 80 --cycles 2 > /dev/null 2>&1
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launch_cfg1.csv python scripts/profile_cycle.py --dim 2 --level 5 --k 10 --cycles 2 > /dev/null 2>&1
echo done
