#!/bin/bash
for lib in librank1_b200_dev_base.so librank1_b200_dev.so; do
echo "== $lib"
R1_LIB_PATH=paper_2403_01778_b200/$lib timeout 400 python tools/fuzz_probe.py 200 11 solves 2>&1 | grep -v '^   ('
done
