timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider 2>&1 | tail -2
bash scripts/ab_bench.sh "cfg2 cfg1" "TMG_X=1"
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_fused2 --csv python scripts/profile_cycle.py --dim 2 --level 7 --k 100 --bpx --cycles 2 2>/dev/null | grep gpu__time | awk -F'","' '{print $5, $NF}' | cut -c1-150
