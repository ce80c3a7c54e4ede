# group size (lanes per element) at high N
AB_REPS=1 AB_NCUBE=40 python scripts/ab.py 9 9 h99_64 h99_128
AB_REPS=1 AB_NCUBE=40 python scripts/ab.py 8 8 h88_64 h88_128
AB_REPS=1 python scripts/ab.py 7 7 h77_32 h77_64
AB_REPS=1 python scripts/ab.py 6 6 h66_32 h66_64
