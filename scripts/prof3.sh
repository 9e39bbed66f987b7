timeout 900 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/t.log 2>&1
bash scripts/ab_bench.sh "cfg1 cfg2 cfg3 cfg5" "TMG_PDL=0 TMG_PDL=1" 2>&1 | grep -v "^ \|Traceback\|json"
tail -1 gpurun_out/t.log
