# per-kernel launch list (ncu duration + dram bytes) of one config, merge on/off
CFG=${CFG:-C2}
for M in 1 0; do
R1_SWEEP_MERGE=$M ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/list_${CFG}_m$M.csv python tools/sweep_probe.py $CFG --reps 2 --warm-ms 1 > /dev/null 2>&1
done
ls -la gpurun_out/list_*
