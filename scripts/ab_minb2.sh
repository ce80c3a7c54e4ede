AB_REPS=1 AB_NCUBE=40 python scripts/ab.py 9 9 mb99_4 mb99_3
AB_REPS=1 AB_NCUBE=40 python scripts/ab.py 8 8 mb88_4 mb88_3
AB_REPS=1 python scripts/ab.py 6 6 mb66_4 mb66_3
AB_REPS=1 python scripts/ab.py 7 7 mb77_4 mb77_3
