#!/bin/bash
timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 600 python tools/c1_probe.py C1 2>&1 | tail -4
timeout 600 python tools/solve_probe.py C5 C2 --alg hoscf --reps 2 2>&1 | grep -v '   it'
