timeout 900 python -m pytest tests/test_bk_gpu.py -q -x 2>&1 | tail -2
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bk_launches4.csv python tools/bk_probe.py 3000 6500 > gpurun_out/bk_ncu.log 2>&1; tail -1 gpurun_out/bk_ncu.log
for v in 1 0 1 0; do R1_BK_UPDATE_DFMA=$v timeout 300 python tools/solve_probe.py C2 C5 --alg ihoscf 2>&1 | grep rep1 | sed "s/^/dfma=$v /"; done
