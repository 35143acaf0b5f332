timeout 900 python -m pytest tests/test_fullsize_gpu.py -q -x -k "c4_solve" 2>&1 | tail -3
