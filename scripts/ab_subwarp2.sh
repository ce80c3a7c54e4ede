AB_REPS=1 python scripts/ab.py 1 1 g11_8_1 g11_4_1 g11_8_2
AB_REPS=1 python scripts/ab.py 2 2 g22_8_1 g22_4_1 g22_8_2
AB_REPS=1 python scripts/ab.py 3 3 g33_8_1 g33_4_1
AB_REPS=1 python scripts/ab.py 4 4 g44_16_1 g44_8_1 g44_8_2
AB_REPS=1 python scripts/ab.py 5 5 g55_32_1 g55_8_1
