set -x
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -5
timeout 900 python bench.py > gpurun_out/r01_bench.json 2> gpurun_out/r01_bench.err; tail -c 3000 gpurun_out/r01_bench.json
CMD="python bench.py --steps 3 --warmup 3 --skip-solve --skip-cpu --skip-configs --e2e-steps 1"
$CMD > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r01_launches.csv $CMD > gpurun_out/ncu_list.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:sweep3_box -s 3 -c 1 -o gpurun_out/r01_sweep_c2 -f $CMD > gpurun_out/ncu_full.log 2>&1; tail -2 gpurun_out/ncu_full.log
