timeout 900 python -m pytest tests/test_gpu_pyramid.py tests/test_gpu_fast_policies.py -q -p no:cacheprovider > gpurun_out/t.log 2>&1
for a in "--dim 3 --level 5 --k 20" "--dim 2 --level 7 --k 100 --bpx" "--dim 2 --level 5 --k 10"; do
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_up_coop" --csv python scripts/profile_cycle.py $a --cycles 2 2>/dev/null | grep gpu__time | awk -F'","' '{print $5, $NF}' | sed "s/.*,//" | tail -1 | sed "s#^#$a #"
done
tail -1 gpurun_out/t.log
