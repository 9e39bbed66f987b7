ncu --set full --import-source on --clock-control none -k regex:"k_amr_residual" -s 0 -c 1 -o gpurun_out/amrres python scripts/amr_cycle.py 2 > /dev/null 2>&1
echo done
