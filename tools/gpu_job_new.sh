set -x
timeout 900 python -m pytest tests/test_bk_gpu.py tests/test_solver_gpu.py -q -x 2>&1 | tail -15
R1_BK_TRACE=1 timeout 300 python tools/bk_probe.py 1000 6500 2>&1 | tail -6
timeout 300 python tools/bk_probe.py 2>&1 | tail -6
timeout 600 python tools/solve_probe.py C2 C4 C5 --alg ihoscf --reps 2 2>&1 | grep -v "^   it"
