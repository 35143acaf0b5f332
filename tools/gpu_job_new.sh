timeout 600 python -m pytest tests/test_bk_gpu.py -q -x -k large_n 2>&1 | tail -3
