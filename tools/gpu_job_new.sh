#!/bin/bash
# decide tolerance A/B in the HOSCF chain (development build)
export R1_LIB_PATH=$PWD/paper_2403_01778_b200/librank1_b200_dev.so
for T in 1e-4 1e-3 1e-2 1e-1; do
  echo "== R1_EIG_DECIDE_TOL=$T =="
  R1_EIG_DECIDE_TOL=$T timeout 600 python tools/decide_probe.py 2>&1 | grep '"cfg": [13]'
done
