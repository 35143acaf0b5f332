timeout 600 python tools/stress_probe.py 20 2>&1 | tail -3
