#!/bin/bash
# two-lane sweep: parity + A/B on the development build (R1_SWEEP_FORK=0/1)
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
export R1_LIB_PATH=$PWD/paper_2403_01778_b200/librank1_b200_dev.so
for F in 0 1 0 1; do
  echo "== FORK=$F =="
  R1_SWEEP_FORK=$F timeout 600 python tools/sweep_probe.py C3 C4 20x20x20x20 128x128x2000 --reps 20 2>&1 | grep -v "CTAs" | grep "median" | sed 's/plan={.*} median/median/'
done
for F in 0 1; do
  echo "== solves FORK=$F =="
  R1_SWEEP_FORK=$F timeout 600 python tools/decide_probe.py 2>&1 | tail -8
done
