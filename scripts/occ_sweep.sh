for b in 4 3 2 1; do echo "blocks/SM=$b"; BBWADG_BLOCKS_PER_SM=$b AB_REPS=1 python scripts/ab.py 7 4 f74 2>&1 | tail -1; done
