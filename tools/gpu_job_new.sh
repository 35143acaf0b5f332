set -x
timeout 900 python -m pytest tests/test_distributed_gpu.py -q -x 2>&1 | tail -15
