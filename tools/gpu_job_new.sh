timeout 900 python -m pytest tests/test_bk_gpu.py tests/test_solver_gpu.py tests/test_solver_props_gpu.py tests/test_fullsize_gpu.py -q 2>&1 | tail -2
