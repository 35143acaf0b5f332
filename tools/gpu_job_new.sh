#!/bin/bash
for i in 1 2; do
for cfg in "R1_SWEEP_DYN_FRAC=0.25" "R1_SWEEP_DYN_FRAC=0.12" "R1_SWEEP_DYN_FRAC=0.4" "R1_SWEEP_DYN_CHUNK=4" "R1_SWEEP_DYN_CHUNK=16"; do
echo "== $cfg"; env $cfg timeout 300 python tools/sweep_probe.py C2 C3 C5 --reps 20 2>&1 | grep -v "^   [a-z]" | sed 's/dims=.*median/median/'
done
done
