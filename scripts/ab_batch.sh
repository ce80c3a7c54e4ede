# batch of library A/B comparisons (see scripts/ab.py)
AB_REPS=1 python scripts/ab.py 7 4 j74 p74 o74
AB_REPS=1 AB_NCUBE=40 python scripts/ab.py 9 9 l99 p99
AB_REPS=1 python scripts/ab.py 1 1 e11_4 e11_8 e11_16
AB_REPS=1 python scripts/ab.py 2 2 e22_4 e22_8
AB_REPS=1 python scripts/ab.py 3 3 e33_2 e33_4
AB_REPS=1 python scripts/ab.py 4 4 e44_2 e44_4
