# sweep parity + timings + launch lists C3/C4
set -x
timeout 900 python -m pytest tests/test_sweep_gpu.py -q -x 2>&1 | tail -3
timeout 600 python tools/sweep_probe.py 2>&1 | grep -v CTAs | tail -12
for C in C3 C4; do
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/list_$C.csv python tools/sweep_probe.py $C --reps 2 --warm-ms 1 > /dev/null 2>&1
done
