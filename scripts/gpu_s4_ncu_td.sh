# session 4: ncu --set full of the finest-level top-downs (adaptive cfg4, exact 243^3)
mkdir -p gpurun_out/s4
ncu --set full --clock-control none --import-source on -k regex:k_amr_topdown -s 6 -c 1 -o gpurun_out/s4/amr_td python scripts/amr_cycle.py 1 fast > gpurun_out/s4/ncu_amr_td.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_topdown -s 4 -c 1 -o gpurun_out/s4/exact_td python scripts/profile_cycle.py --precision exact --cycles 1 > gpurun_out/s4/ncu_exact_td.log 2>&1
ls -la gpurun_out/s4
