# full GPU test suite (no -x: report every failure)
set -x
timeout 2400 python -m pytest tests -m gpu -q --durations=20 2>&1 | tail -60
