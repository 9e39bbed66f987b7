# profiles of the current build: cfg5 launch list (2 cycles) and a --set full capture of the fused pass at 729^3
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launch_cfg5.csv python scripts/profile_cycle.py --dim 3 --level 6 --k 80 --cycles 2 > /dev/null 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_fused3 -s 1 -c 1 -o gpurun_out/fused3_729 python scripts/profile_cycle.py --dim 3 --level 6 --k 80 --cycles 2 > /dev/null 2>&1
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launch_cfg4.csv python scripts/amr_cycle.py 2 > /dev/null 2>&1
echo done
