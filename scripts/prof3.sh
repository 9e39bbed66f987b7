timeout 900 python -m pytest tests/test_gpu_pyramid.py tests/test_gpu_slabs.py tests/test_gpu_fast_policies.py -q -p no:cacheprovider 2>&1 | tail -1
for a in "--dim 3 --level 5 --k 20" "--dim 3 --level 6 --k 80" "--dim 2 --level 7 --k 100 --bpx"; do
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_combine" --csv python scripts/profile_cycle.py $a --cycles 2 2>/dev/null | grep gpu__time | awk -F'","' '{print $5, $NF}' | sed "s/.*,//" | tail -1
done
