bash scripts/ab_bench.sh "cfg5 cfg3 cfg2" "TMG_GRID_CAP=32 TMG_GRID_CAP=8 TMG_GRID_CAP=16 TMG_GRID_CAP=64" 2>&1 | grep -v "^ \|Traceback\|json"
