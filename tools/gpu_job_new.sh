#!/bin/bash
# soak at HEAD (release library): mixed sweeps + solves, short processes
for S in 101 102 103 104 105 106 107 108; do
    timeout 200 python tools/fuzz_probe.py 30 $S 2>&1 | grep "FAILED\|fuzz:\|error" | cut -c1-200
done
timeout 200 python tools/bk_fuzz_probe.py 40 9 2>&1 | tail -1 | cut -c1-200
