bash scripts/ab_bench.sh "cfg5 cfg3" "TMG_X=1 TMG_LIB=./var_stream.so TMG_X=2 TMG_LIB=./var_stream.so" 2>&1 | grep -v "^ \|Traceback\|json"
