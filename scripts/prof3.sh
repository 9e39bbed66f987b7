timeout 900 python -m pytest tests/test_gpu_pyramid.py tests/test_gpu_slabs.py -q -p no:cacheprovider 2>&1 | tail -1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_topdown_tri" --csv python scripts/profile_cycle.py --dim 3 --level 6 --k 80 --cycles 2 2>/dev/null | grep gpu__time | awk -F'","' '{print $5, $NF}' | sed "s/.*,//" | tail -2
