#!/bin/bash
export R1_LIB_PATH=paper_2403_01778_b200/librank1_b200_dev.so
for nc in 148 140 132 120; do
echo "== ncta $nc"
R1_SWEEP_NCTA=$nc timeout 300 python tools/sweep_probe.py C5 C2 --reps 20 --warm-ms 200 2>&1 | grep -o 'level-0.*\|median.*'
done
