# ncu --set full of the 2D fused pass at 2187^2 (cfg2, BPX)
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:k_fused2 -s 1 -c 1 -o gpurun_out/f2 python scripts/profile_cycle.py --dim 2 --level 7 --k 100 --bpx --cycles 2 > gpurun_out/ncu_f2.log 2>&1
python scripts/summarize_ncu.py full gpurun_out/f2.ncu-rep
python scripts/ncu_lines.py gpurun_out/f2.ncu-rep 25
ncu -i gpurun_out/f2.ncu-rep --page raw --csv 2>/dev/null | python3 -c "
import csv,sys
rows=list(csv.reader(sys.stdin)); hdr,units,vals=rows[0],rows[1],rows[2]
for i,h in enumerate(hdr):
    if ('average_warps_issue_stalled' in h and 'per_issue_active' in h) or 'achieved_occupancy' in h or 'sm__warps_active' in h or 'dram__throughput' in h:
        try:
            if float(vals[i].replace(',',''))>0.05: print(h, vals[i])
        except: pass
"
