# sub-warp element groups (TG = 8 / 16) vs whole-warp groups with ET elements per lane, low N
AB_REPS=1 python scripts/ab.py 1 1 g11_32_4 g11_16_1 g11_8_1
AB_REPS=1 python scripts/ab.py 2 2 g22_32_4 g22_16_1 g22_8_1
AB_REPS=1 python scripts/ab.py 3 3 g33_32_2 g33_16_1 g33_8_1
AB_REPS=1 python scripts/ab.py 4 4 g44_32_2 g44_16_1
AB_REPS=1 python scripts/ab.py 5 5 g55_32_1 g55_16_1
