timeout 120 python tools/c1_probe.py C1 2>&1 | tail -1
timeout 120 python tools/c1_probe.py C4 2>&1 | tail -1
timeout 200 python tools/solve_probe.py C2 C3 C5 --alg hoscf,ihoscf 2>&1 | grep rep1
R1_DEBUG_EIG=1 timeout 120 python tools/c1_probe.py C1 2>&1 | grep "r1 eig" | sed -n '150,151p'
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
