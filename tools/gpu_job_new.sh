timeout 900 python -m pytest tests/test_bk_gpu.py tests/test_solver_gpu.py -q -x 2>&1 | tail -2
R1_BK_TRACE=1 timeout 300 python tools/bk_probe.py 3000 2>&1 | grep "r1 bk" | tail -1
