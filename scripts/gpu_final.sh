# round-2 evidence: bench lines of every workload, launch lists, ncu --set full of the 2D pass
mkdir -p gpurun_out/final
O=gpurun_out/final
timeout 600 python bench.py > $O/bench_cfg5.json 2> $O/bench_cfg5.err; echo cfg5=$?
for w in cfg3 cfg2 cfg1; do timeout 300 python bench.py --workload $w --no-cpu-baseline > $O/bench_$w.json 2> $O/bench_$w.err; done
timeout 300 python bench.py --workload cfg4 --no-cpu-baseline > $O/bench_cfg4_fast.json 2> $O/bench_cfg4_fast.err
timeout 300 python bench.py --workload cfg4 --precision exact --no-cpu-baseline > $O/bench_cfg4_exact.json 2> $O/bench_cfg4_exact.err
timeout 300 python bench.py --precision fast-complex64 --no-cpu-baseline > $O/bench_cfg5_c64.json 2> $O/bench_cfg5_c64.err
for f in $O/bench_*.json; do python -c "
import json,sys; d=json.load(open('$f')); r=d.get('roofline',{}); print('$f', round(d['value']/1e9,3), 'G', round(d['ms_per_step'],4), 'ms frac', round(r.get('frac',0),3), 'moved', round(r.get('frac_moved_basis',0) or 0,3), 'e2e', round(d['e2e']['value']/1e9,3), 'clk', d['clocks']['sm_mhz'], d['clocks']['reasons'])" 2>/dev/null || echo "$f failed"; done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
ncu --metrics $M --clock-control none --csv --log-file $O/launch_cfg2.csv python scripts/profile_cycle.py --dim 2 --level 7 --k 100 --bpx --cycles 2 > /dev/null 2>&1
ncu --metrics $M --clock-control none --csv --log-file $O/launch_cfg1.csv python scripts/profile_cycle.py --dim 2 --level 5 --k 10 --cycles 2 > /dev/null 2>&1
ncu --metrics $M --clock-control none --csv --log-file $O/launch_cfg4_fast.csv python scripts/amr_cycle.py 2 fast > /dev/null 2>&1
ncu --metrics $M --clock-control none --csv --log-file $O/launch_cfg4_exact.csv python scripts/amr_cycle.py 2 exact > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_fused2 -s 1 -c 1 -o $O/f2_final python scripts/profile_cycle.py --dim 2 --level 7 --k 100 --bpx --cycles 2 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_amr_residual -c 1 -o $O/amr_res_fast python scripts/amr_cycle.py 1 fast > /dev/null 2>&1
ls $O
