#!/bin/bash
mkdir -p gpurun_out
export R1_LIB_PATH=paper_2403_01778_b200/librank1_b200_dev.so
export R1_EIG_TMA=0
for ce in "8 8" "4 4" "2 4" "4 2" ; do set -- $ce
echo "== check $1 min $2"
R1_EIG_CHECK=$1 R1_EIG_MIN_STEPS=$2 R1_DEBUG_EIG=1 timeout 300 python tools/eig_debug_probe.py C5 2>&1 | tail -4
R1_EIG_CHECK=$1 R1_EIG_MIN_STEPS=$2 R1_DEBUG_EIG=1 timeout 300 python tools/eig_debug_probe.py C2 2>&1 | tail -2
done
R1_DEBUG_EIG_TEXT=1 timeout 300 python tools/eig_debug_probe.py C5 2>&1 | grep t_extremes | tail -3
