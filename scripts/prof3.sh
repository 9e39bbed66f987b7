timeout 900 python -m pytest tests/test_gpu_slabs.py tests/test_gpu_fast_policies.py tests/test_gpu_pyramid.py -q -p no:cacheprovider > gpurun_out/t.log 2>&1
bash scripts/ab_bench.sh "cfg3" "TMG_X=1 TMG_ZCHUNKS=8 TMG_X=2" 2>&1 | grep -v "^ \|Traceback\|json"
tail -1 gpurun_out/t.log; grep FAILED gpurun_out/t.log | head -5
