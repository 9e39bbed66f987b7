timeout 900 python -m pytest tests/test_gpu_amr.py tests/test_gpu_dynamic.py -q -p no:cacheprovider 2>&1 | tail -1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_amr" --csv python scripts/amr_cycle.py 2 2>/dev/null | grep gpu__time | awk -F'","' '{print $5, $NF}' | cut -c1-100 | tail -17
