#!/bin/bash
R1_SWEEP_W8=1 R1_SWEEP_STAGE_REGS=0 timeout 600 python -m pytest tests/test_sweep_gpu.py -q -x 2>&1 | tail -2
for i in 1 2; do
for cfg in "R1_SWEEP_W8=0" "R1_SWEEP_W8=1 R1_SWEEP_STAGE_REGS=0" "R1_SWEEP_W8=1"; do
echo "== $cfg"; env $cfg timeout 300 python tools/sweep_probe.py C2 C5 C1 --reps 20 2>&1 | grep -v "^   [a-z]" | sed 's/dims=.*median/median/'
done
done
