# ncu --set full of the cfg4 finest-level top-down and residual (first cycle)
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:k_amr_topdown -s 6 -c 1 -o gpurun_out/amr_td python scripts/amr_cycle.py 1 > gpurun_out/ncu_amr_td.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_amr_residual -c 1 -o gpurun_out/amr_res python scripts/amr_cycle.py 1 > gpurun_out/ncu_amr_res.log 2>&1
for r in amr_td amr_res; do python scripts/summarize_ncu.py full gpurun_out/$r.ncu-rep; python scripts/ncu_lines.py gpurun_out/$r.ncu-rep 16; done
