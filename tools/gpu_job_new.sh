timeout 600 python -m pytest tests/test_solver_props_gpu.py tests/test_solver_gpu.py tests/test_baselines_gpu.py -q 2>&1 | grep -E "passed|failed|^E " | head -20
