# one ncu --set full capture of the finest-level fused AMR kernel (cfg4)
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:k_amr_fused_fine -c 1 -o gpurun_out/amr_fused ${NCU_EXTRA} python scripts/amr_cycle.py 1 > gpurun_out/ncu_amr.log 2>&1
tail -3 gpurun_out/ncu_amr.log
python scripts/summarize_ncu.py full gpurun_out/amr_fused.ncu-rep
python scripts/ncu_lines.py gpurun_out/amr_fused.ncu-rep 30
