timeout 900 python -m pytest tests/test_gpu_amr.py tests/test_gpu_dynamic.py tests/test_gpu_goldens.py -q -p no:cacheprovider > gpurun_out/t.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_amr_topdown" --csv python scripts/amr_cycle.py 2 2>/dev/null | grep gpu__time | awk -F'","' '{print $5, $NF}' | sed "s/.*,//" | tail -1
timeout 300 python bench.py --workload cfg4 --no-cpu-baseline --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg4', d['value']/1e9, d['ms_per_step'])"
tail -1 gpurun_out/t.log
