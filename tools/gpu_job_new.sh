timeout 900 python -m pytest tests/test_fullsize_gpu.py -q -k "c3_fixed" 2>&1 | tail -3
