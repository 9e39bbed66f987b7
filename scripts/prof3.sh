timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider 2>&1 | tail -1
ncu --set full --import-source on --clock-control none -k regex:k_fused2 -s 1 -c 1 -o gpurun_out/fused2b_full python scripts/profile_cycle.py --dim 2 --level 7 --k 100 --bpx --cycles 3 > /dev/null 2>&1
