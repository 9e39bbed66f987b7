bash scripts/ab_bench.sh "cfg3" "TMG_LIB=./var_ty4.so TMG_ZCHUNKS=4 TMG_ZCHUNKS=6" 2>&1 | grep -v "^ \|Traceback\|json"
for z in 4 5 6 7 8; do TMG_LIB=./var_ty4.so TMG_ZCHUNKS=$z python bench.py --workload cfg3 --no-cpu-baseline --steps 10 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('ty4 z$z', round(d['value']/1e9,2), round(d['ms_per_step'],4), round(d['fine_pass_ms'],4))"; done
