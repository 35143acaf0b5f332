timeout 600 python -m pytest tests/test_bk_gpu.py -q 2>&1 | tail -1
R1_BK_TRACE=1 timeout 300 python tools/bk_probe.py 6500 2>&1 | tail -3
timeout 600 python tools/solve_probe.py C2 C5 --alg ihoscf --reps 2 2>&1 | grep rep1
