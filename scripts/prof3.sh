TMG_LC_DBG=48 python scripts/profile_cycle.py --dim 3 --level 5 --k 20 --cycles 1 2>&1 | sort | head -60
