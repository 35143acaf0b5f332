timeout 900 python -m pytest tests/test_dev_switches_gpu.py tests/test_bk_gpu.py -q 2>&1 | tail -15
