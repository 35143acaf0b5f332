R1_DEBUG_EIG_TEXT=1 timeout 120 python tools/c1_probe.py C1 2>&1 | grep "t_extremes" | sed -n '500,503p'
timeout 120 python tools/c1_probe.py C1 2>&1 | tail -1
timeout 300 python tools/solve_probe.py C3 C2 C5 --alg hoscf --reps 2 2>&1 | grep rep1
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -2
