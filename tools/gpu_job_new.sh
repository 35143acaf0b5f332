timeout 300 python tools/solve_probe.py C5 --alg ihoscf --reps 1 2>&1 | tail -6
R1_RQI_CUSOLVER=1 timeout 300 python tools/solve_probe.py C5 --alg ihoscf --reps 1 2>&1 | tail -6
