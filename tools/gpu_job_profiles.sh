# Round-end evidence: bench line, launch lists and ncu captures (read back with
# tools/ncu_summary.py / tools/ncu_kernel_summary.py into profiles/).
set -x
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/r01_bench.json 2> gpurun_out/r01_bench.err; tail -c 300 gpurun_out/r01_bench.err
CMD="python bench.py --steps 3 --warmup 3 --skip-solve --skip-cpu --skip-configs --e2e-steps 1"
$CMD > gpurun_out/plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r01_launches.csv $CMD > gpurun_out/ncu_list.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep3_box -s 3 -c 1 -o gpurun_out/r01_sweep_c2 -f $CMD > gpurun_out/ncu_full.log 2>&1; tail -1 gpurun_out/ncu_full.log
timeout 600 python tools/solve_probe.py C2 --alg ihoscf --reps 1 > gpurun_out/rqi_plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01_launches_rqi_c2.csv python tools/solve_probe.py C2 --alg ihoscf --reps 1 > gpurun_out/rqi_ncu.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:bk_panel_smem -s 20 -c 1 -o gpurun_out/r01_bk_panel -f python tools/bk_probe.py 3000 > gpurun_out/bk_full.log 2>&1; tail -1 gpurun_out/bk_full.log
timeout 600 python tools/c1_probe.py C1 > gpurun_out/c1_plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01_launches_c1.csv python tools/c1_probe.py C1 > gpurun_out/c1_ncu.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:lanczos_cluster -s 50 -c 1 -o gpurun_out/r01_lanczos_cluster -f python tools/c1_probe.py C1 > gpurun_out/lz_full.log 2>&1; tail -1 gpurun_out/lz_full.log
C3CMD="python tools/sweep_probe.py C3 --reps 2 --warm-ms 0"
$C3CMD > gpurun_out/c3_plain.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r01_launches_c3.csv $C3CMD > gpurun_out/c3_ncu_list.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep3_box -s 0 -c 1 -o gpurun_out/r01_sweep_c3 -f $C3CMD > gpurun_out/c3_full.log 2>&1; tail -1 gpurun_out/c3_full.log
