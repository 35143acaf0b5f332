#!/bin/bash
timeout 900 python -m pytest tests/test_sweep_gpu.py tests/test_fuzz_gpu.py -q -x 2>&1 | tail -2
for S in 71 72 73; do timeout 200 python tools/fuzz_probe.py 30 $S sweeps 2>&1 | grep "FAILED\|fuzz:\|error" | cut -c1-200; done
timeout 300 python tools/fork_fuzz_probe.py 100 9 2>&1 | tail -1 | cut -c1-200
timeout 300 python tools/sweep_probe.py C4 C3 40x40x40x40 16x16x16x16x16 10x10x10x10x10x10 60x60x60x60 --reps 30 2>&1 | grep "median" | sed 's/plan={.*} median/median/'
timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 300 python tools/fuzz_probe.py 60 15 hoscf 2>&1 | tail -2 | cut -c1-200
