set -x
timeout 900 python -m pytest tests/test_greedy_io_gpu.py tests/test_cpp_dropin.py tests/test_baselines_gpu.py -q -x 2>&1 | tail -25
