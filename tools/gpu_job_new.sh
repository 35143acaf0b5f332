set -x
timeout 1200 python -m pytest tests/test_fullsize_gpu.py -q -x --durations=10 2>&1 | tail -15
