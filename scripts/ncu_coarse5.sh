# ncu --set full of the non-fused kernels of the 729^3 cycle (combine, level-5 top-down, restriction)
mkdir -p gpurun_out
for k in k_combine k_topdown_tri k_restrict; do
ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o gpurun_out/c5_$k python scripts/profile_cycle.py --dim 3 --level 6 --k 80 --cycles 2 > /dev/null 2>&1
python scripts/summarize_ncu.py full gpurun_out/c5_$k.ncu-rep
python scripts/ncu_lines.py gpurun_out/c5_$k.ncu-rep 8
done
