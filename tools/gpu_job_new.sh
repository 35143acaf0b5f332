timeout 60 python tools/c1_probe.py C1 2>&1 | tail -1
R1_DEBUG_EIG=1 timeout 60 python tools/c1_probe.py C1 2>&1 | grep "r1 eig" > gpurun_out/c1_eig_dbg.txt
timeout 120 python tools/solve_probe.py C3 --alg hoscf --reps 2 2>&1 | grep rep1 | cut -c1-150
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
