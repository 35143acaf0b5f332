#!/bin/bash
# evidence after the wide shapes: bench line, launch list, --set full captures (C5 sweep, C3 level 0)
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r02_bench_wide.log 2>&1; tail -c 600 gpurun_out/r02_bench_wide.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches_c5_wide.csv python bench.py --steps 3 --warmup 3 --skip-configs --skip-cpu --skip-solve > gpurun_out/ncu_list.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'sweep3_box|finish_kernel' -s 8 -c 2 -o gpurun_out/sw_c5_wide -f python tools/sweep_probe.py C5 --reps 3 --warm-ms 50 > gpurun_out/ncu_c5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'sweep3_box|finish_kernel|finish_b01' -s 16 -c 8 -o gpurun_out/sw_c3_wide -f python tools/sweep_probe.py C3 --reps 3 --warm-ms 50 > gpurun_out/ncu_c3.log 2>&1
tail -2 gpurun_out/ncu_c5.log gpurun_out/ncu_c3.log
ls -la gpurun_out
