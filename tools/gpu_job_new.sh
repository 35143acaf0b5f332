#!/bin/bash
# confirm: sweep fuzz in short processes on the RELEASE library (PDL off), then PDL on with the failing seed repeated
for S in 11 21 31 41 51 61 71 81 91 101 111 121; do
    echo "== release seed=$S =="
    timeout 200 python tools/fuzz_probe.py 35 $S 2>&1 | grep "FAILED\|fuzz:\|error" | cut -c1-200
done
export R1_LIB_PATH=$PWD/paper_2403_01778_b200/librank1_b200_dev.so
for S in 51 51 51 52 53 54; do
    echo "== dev PDL=1 seed=$S =="
    R1_SWEEP_PDL=1 timeout 200 python tools/fuzz_probe.py 35 $S 2>&1 | grep "FAILED\|fuzz:\|error" | cut -c1-200
done
