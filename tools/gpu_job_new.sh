R1_DEBUG_EIG=1 timeout 120 python tools/solve_probe.py C2 C5 --alg hoscf --reps 1 2>&1 | grep "r1 eig" | sed 's/lo=.*res_hi=[^ ]* //' | head -12
