timeout 900 python -m pytest tests/test_gpu_pyramid.py tests/test_gpu_slabs.py -q -p no:cacheprovider 2>&1 | grep -E "passed|failed|FAILED|Error" | head
bash scripts/ab_bench.sh "cfg2 cfg3 cfg1 cfg5" "TMG_UP=0 TMG_UP=1"
bash scripts/ab_bench.sh "cfg5" "TMG_TRI_COARSE=0"
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launch_cfg2.csv python scripts/profile_cycle.py --dim 2 --level 7 --k 100 --bpx --cycles 2 > gpurun_out/ncu_cfg2.log 2>&1
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launch_cfg3.csv python scripts/profile_cycle.py --dim 3 --level 5 --k 20 --cycles 2 > gpurun_out/ncu_cfg3.log 2>&1
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launch_cfg5.csv python scripts/profile_cycle.py --dim 3 --level 6 --k 80 --cycles 2 > gpurun_out/ncu_cfg5.log 2>&1
ncu --metrics $M --clock-control none --csv --log-file gpurun_out/launch_cfg1.csv python scripts/profile_cycle.py --dim 2 --level 5 --k 10 --cycles 2 > gpurun_out/ncu_cfg1.log 2>&1
