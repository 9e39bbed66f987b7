# ncu --set full of the fused 3D pass at 243^3 (one launch) with SASS-level source counters
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:k_fused3_r2 -s 1 -c 1 -o gpurun_out/f3_243 python scripts/profile_cycle.py --dim 3 --level 5 --k 20 --cycles 2 > gpurun_out/ncu_f3.log 2>&1
python scripts/summarize_ncu.py full gpurun_out/f3_243.ncu-rep
