AB_REPS=2 python scripts/ab.py 7 4 t74_128 t74_64 t74_256
AB_REPS=1 python scripts/ab.py 5 3 t53_128 t53_64
