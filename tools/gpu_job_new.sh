#!/bin/bash
# dynamic-tail share / chunk with the wide shapes (development build)
export R1_LIB_PATH=$PWD/paper_2403_01778_b200/librank1_b200_dev.so
for F in 0.25 0.15 0.35 0.25; do
 for C in 8 4 16; do
  echo "== FRAC=$F CHUNK=$C =="
  R1_SWEEP_DYN_FRAC=$F R1_SWEEP_DYN_CHUNK=$C timeout 300 python tools/sweep_probe.py C5 C2 C3 --reps 20 2>&1 | grep "median" | sed 's/plan={.*nseg.: \([0-9]*\).*} median/nseg \1 median/'
 done
done
