# ncu --set full of the top-level sweep kernel for one config, merge on/off
set -x
CFG=${CFG:-C2}
python tools/sweep_probe.py $CFG --reps 3 --warm-ms 50 > gpurun_out/ncu_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sweep3_box -s 4 -c 1 -o gpurun_out/sw_${CFG}_merge -f python tools/sweep_probe.py $CFG --reps 3 --warm-ms 50 > gpurun_out/ncu1.log 2>&1
R1_SWEEP_MERGE=0 ncu --set full --clock-control none --import-source on -k regex:sweep3_box -s 4 -c 1 -o gpurun_out/sw_${CFG}_nomerge -f python tools/sweep_probe.py $CFG --reps 3 --warm-ms 50 > gpurun_out/ncu2.log 2>&1
tail -3 gpurun_out/ncu1.log gpurun_out/ncu2.log
