#!/bin/bash
# BK panel: factorisation time vs size and forced cluster size, phase trace
mkdir -p gpurun_out
export R1_LIB_PATH=$PWD/paper_2403_01778_b200/librank1_b200_dev.so
python tools/bk_time_probe.py 600 1500 3000 6500
for g in 1 2 4 8 12 16; do R1_BK_G=$g python tools/bk_time_probe.py 600 1500 3000 2>&1 | grep -v Error; done
R1_BK_TRACE=1 REPS=1 python tools/bk_time_probe.py 600 3000 6500 2>&1
for g in 1 2 4 16; do R1_BK_G=$g R1_BK_TRACE=1 REPS=1 python tools/bk_time_probe.py 600 2>&1; done
