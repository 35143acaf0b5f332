timeout 600 python -m pytest tests/test_bk_gpu.py tests/test_solver_gpu.py -q -x 2>&1 | tail -1
for v in old new old new; do R1_LIB_PATH=$PWD/abtest/$v.so timeout 120 python tools/solve_probe.py C2 C5 --alg ihoscf 2>&1 | grep rep1 | sed "s/^/$v /" | cut -c1-70; done
R1_BK_TRACE=1 timeout 120 python tools/bk_probe.py 3000 2>&1 | grep "r1 bk" | tail -1
