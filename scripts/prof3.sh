timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider -k "2 or fused" > gpurun_out/t.log 2>&1
bash scripts/ab_bench.sh "cfg2 cfg1" "TMG_X=1" 2>&1 | grep -v "^ \|Traceback\|json"
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_fused2" --csv python scripts/profile_cycle.py --dim 2 --level 7 --k 100 --bpx --cycles 2 2>/dev/null | grep gpu__time | awk -F'","' '{print $5, $NF}' | sed "s/.*,//" | tail -1
tail -1 gpurun_out/t.log
