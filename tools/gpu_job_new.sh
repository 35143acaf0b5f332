#!/bin/bash
export R1_LIB_PATH=$PWD/paper_2403_01778_b200/librank1_b200_dev.so
for S in 51 52 53 54 55 56 57 58 59 60 61 62 63 64 65 66; do
  echo "== PDL=1 sweeps only seed=$S =="
  R1_SWEEP_PDL=1 timeout 200 python tools/fuzz_probe.py 30 $S sweeps 2>&1 | grep "FAILED\|fuzz:\|error" | cut -c1-160
done
