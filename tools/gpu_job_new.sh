for g in 148 96 64 48 32; do R1_EIG_GRID=$g timeout 120 python tools/solve_probe.py C2 C5 --alg hoscf --reps 3 2>&1 | grep rep2 | sed "s/^/G=$g /" | cut -c1-140; done
