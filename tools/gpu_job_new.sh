#!/bin/bash
for rep in 1 2; do for lib in librank1_b200_dev_base.so librank1_b200_dev.so; do
echo "== $lib"
R1_LIB_PATH=paper_2403_01778_b200/$lib timeout 300 python tools/sweep_probe.py C4 C3 --reps 30 --warm-ms 300 2>&1 | grep -o 'C[0-9] dims.*median.*' | sed 's/plan=.*median/median/'
done; done
