AB_REPS=1 python scripts/ab.py 7 4 j74 l74
AB_REPS=1 AB_NCUBE=40 python scripts/ab.py 9 9 m99 l99
