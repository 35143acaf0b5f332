#!/bin/bash
timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for S in 11 21 31 41; do timeout 200 python tools/fuzz_probe.py 30 $S 2>&1 | grep "FAILED\|fuzz:\|error" | cut -c1-200; done
timeout 300 python tools/fuzz_probe.py 90 14 hoscf 2>&1 | tail -2 | cut -c1-200
timeout 200 python tools/decide_probe.py 2>&1 | tail -6 | cut -c1-200
