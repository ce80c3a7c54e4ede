AB_REPS=2 python scripts/ab.py 7 4 ref74 stcs74
AB_REPS=1 python scripts/ab.py 5 3 nost53 stcs53
bash scripts/gpu_dram_ab.sh ref74 stcs74 2>&1 | grep -v "N=7"
