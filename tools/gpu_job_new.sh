#!/bin/bash
export R1_LIB_PATH=$PWD/paper_2403_01778_b200/librank1_b200_dev.so
for i in 1 2 3; do echo "== PDL=1 fresh plans run $i =="; R1_SWEEP_PDL=1 timeout 120 python tools/pdl_hunt.py 6000 1 2>&1 | tail -1; done
for i in 1 2; do echo "== PDL=1 cached plans run $i =="; R1_SWEEP_PDL=1 timeout 120 python tools/pdl_hunt.py 6000 0 2>&1 | tail -1; done
echo "== PDL=1 WIDE=0 fresh =="; R1_SWEEP_PDL=1 R1_SWEEP_WIDE=0 timeout 120 python tools/pdl_hunt.py 6000 1 2>&1 | tail -1
echo "== PDL=1 WIDE=0 fresh =="; R1_SWEEP_PDL=1 R1_SWEEP_WIDE=0 timeout 120 python tools/pdl_hunt.py 6000 1 2>&1 | tail -1
echo "== PDL=0 fresh =="; R1_SWEEP_PDL=0 timeout 120 python tools/pdl_hunt.py 6000 1 2>&1 | tail -1
