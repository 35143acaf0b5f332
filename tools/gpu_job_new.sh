#!/bin/bash
# PDL sweep chain + self-resetting work counter: parity, then A/B on the development build
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
export R1_LIB_PATH=$PWD/paper_2403_01778_b200/librank1_b200_dev.so
for F in 0 1 0 1; do
  echo "== PDL=$F =="
  R1_SWEEP_PDL=$F timeout 600 python tools/sweep_probe.py C5 C2 C3 C4 C1 --reps 20 2>&1 | grep -v "CTAs" | grep "median" | sed 's/plan={.*} median/median/'
done
for F in 0 1; do
  echo "== solves PDL=$F =="
  R1_SWEEP_PDL=$F timeout 600 python tools/decide_probe.py 2>&1 | tail -6
done
