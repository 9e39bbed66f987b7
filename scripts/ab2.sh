timeout 900 python -m pytest tests/test_gpu_pyramid.py -q -p no:cacheprovider 2>&1 | tail -1
bash scripts/ab_bench.sh "cfg2 cfg1" "TMG_X=1 TMG_LIB=./var_s1200.so" 2>&1 | grep -v "^ \|Traceback\|json"
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_up_coop --csv python scripts/profile_cycle.py --dim 2 --level 7 --k 100 --bpx --cycles 2 2>/dev/null | grep gpu__time | awk -F'","' '{print $5, $NF}' | cut -c1-150
