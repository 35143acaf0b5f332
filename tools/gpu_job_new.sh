timeout 600 python -m pytest tests/test_cpp_dropin.py -q 2>&1 | tail -2
