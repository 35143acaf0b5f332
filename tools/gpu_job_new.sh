#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_sweep_gpu.py tests/test_fullsize_gpu.py -q -x -k "sweep or first or deterministic or c3" 2>&1 | tail -2
for i in 1 2 3; do
for v in old new; do
echo "== $v"; R1_LIB_PATH=abtest/$v/librank1_b200.so timeout 300 python tools/sweep_probe.py C2 C3 C4 C5 --reps 20 2>&1 | grep -v "^   [a-z]" | sed 's/dims=.*median/median/'
done
done
for v in old new; do
R1_LIB_PATH=abtest/$v/librank1_b200.so timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:finish_kernel -c 8 --csv --log-file gpurun_out/fin_$v.csv python tools/sweep_probe.py C2 C3 --reps 2 --warm-ms 0 > /dev/null 2>&1
done
