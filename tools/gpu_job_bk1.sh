#!/bin/bash
# BK panel change check: output hashes (compare with the previous build's) and device time
mkdir -p gpurun_out
python tools/bk_hash_probe.py
python tools/bk_time_probe.py 600 1500 3000 6500
if [ -n "$BK_TRACE" ]; then for c in 1 2 16; do R1_LIB_PATH=$PWD/paper_2403_01778_b200/librank1_b200_dev.so R1_BK_TRACE=$c REPS=1 python tools/bk_time_probe.py 6500 2>&1 | grep 'r1 bk'; done; fi
if [ -n "$BK_TESTS" ]; then timeout 900 python -m pytest tests/test_bk_gpu.py -q -x 2>&1 | tail -2; fi
