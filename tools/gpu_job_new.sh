timeout 900 python -m pytest tests/test_acceptance_gpu.py -q --durations=5 2>&1 | tail -25
