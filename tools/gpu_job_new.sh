#!/bin/bash
for lib in librank1_b200_dev_cu2.so librank1_b200_dev.so; do
export R1_LIB_PATH=paper_2403_01778_b200/$lib
echo "== $lib"
R1_DEBUG_EIG=1 timeout 300 python tools/eig_debug_probe.py C5 2>&1 | tail -4 | cut -c1-330
R1_DEBUG_EIG=1 timeout 300 python tools/eig_debug_probe.py C2 2>&1 | tail -3 | cut -c1-330
done
