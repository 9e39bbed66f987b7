# launch lists for cfg2 (2D L7 BPX) and cfg3, and a full capture of the 2D fused pass
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
python scripts/profile_cycle.py --dim 2 --level 7 --k 100 --bpx --cycles 2 > /dev/null 2>&1 || echo cfg2 run failed
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launch_cfg2.csv python scripts/profile_cycle.py --dim 2 --level 7 --k 100 --bpx --cycles 2 > gpurun_out/ncu_cfg2.log 2>&1
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launch_cfg3.csv python scripts/profile_cycle.py --dim 3 --level 5 --k 20 --cycles 2 > gpurun_out/ncu_cfg3.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_fused2 -s 1 -c 1 -o gpurun_out/fused2_full python scripts/profile_cycle.py --dim 2 --level 7 --k 100 --bpx --cycles 3 > gpurun_out/ncu_f2full.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_combine -s 1 -c 1 -o gpurun_out/combine3_full python scripts/profile_cycle.py --dim 3 --level 5 --k 20 --cycles 3 > gpurun_out/ncu_c3full.log 2>&1
echo done
