timeout 600 python -m pytest tests/test_reference_kats_gpu.py -q 2>&1 | tail -15
