bash scripts/ab_bench.sh "cfg3 cfg2 cfg1 cfg5" "TMG_X=1 TMG_LIB=./var_p64k.so" 2>&1 | grep -v "^ \|Traceback\|json"
