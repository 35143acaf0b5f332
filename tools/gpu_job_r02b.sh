#!/bin/bash
# Round-2 evidence after the tiled Lanczos step: full suite, bench line, C5
# HOSCF launch list, ncu --set full of one warm tiled Lanczos launch (C5) and
# of one C2 launch.
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/r02_bench_c5_lanczos.log 2>&1; tail -c 400 gpurun_out/r02_bench_c5_lanczos.log
P="python tools/solve_probe.py C5 --alg hoscf --reps 1"
$P > gpurun_out/c5_plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_c5_hoscf.csv $P > gpurun_out/c5_ncu_list.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lanczos_kernel -s 4 -c 1 -o gpurun_out/r02_lanczos_tiled_c5 -f $P > gpurun_out/lz_c5_full.log 2>&1; tail -1 gpurun_out/lz_c5_full.log
P2="python tools/solve_probe.py C2 --alg hoscf --reps 1"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lanczos_kernel -s 1 -c 1 -o gpurun_out/r02_lanczos_tiled_c2 -f $P2 > gpurun_out/lz_c2_full.log 2>&1; tail -1 gpurun_out/lz_c2_full.log
