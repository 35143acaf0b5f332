#!/bin/bash
export R1_LIB_PATH=paper_2403_01778_b200/librank1_b200_dev.so
for sm in 1 0; do
echo "== small $sm"
R1_EIG_SMALL=$sm timeout 300 python tools/solve_probe.py C3 --alg hoscf --reps 2 2>&1 | grep -v '   it'
R1_EIG_SMALL=$sm timeout 300 python tools/c1_probe.py C1 2>&1 | tail -1
R1_EIG_SMALL=$sm timeout 300 python tools/c1_probe.py C4 2>&1 | tail -1
done
