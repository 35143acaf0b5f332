timeout 120 python tools/c1_probe.py C1 2>&1 | tail -1
timeout 120 python tools/c1_probe.py C4 2>&1 | tail -1
timeout 200 python tools/solve_probe.py C3 --alg hoscf,ihoscf 2>&1 | grep rep1
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -5
