# launch-bound minimum blocks per SM (register cap) at mid N
AB_REPS=1 python scripts/ab.py 5 5 mb55_4 mb55_5 mb55_6
AB_REPS=1 python scripts/ab.py 5 3 mb53_4 mb53_5 mb53_6
AB_REPS=1 python scripts/ab.py 6 6 mb66_4 mb66_5
AB_REPS=1 python scripts/ab.py 4 4 mb44_4 mb44_5 mb44_6
AB_REPS=1 python scripts/ab.py 3 3 mb33_4 mb33_6 mb33_8
AB_REPS=1 python scripts/ab.py 7 4 mb74_4 mb74_5
