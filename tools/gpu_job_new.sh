timeout 900 python bench.py > gpurun_out/r01_bench.json 2> gpurun_out/r01_bench.err; tail -c 400 gpurun_out/r01_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bk_launches2.csv python tools/bk_probe.py 3000 6500 > gpurun_out/bk_ncu.log 2>&1; tail -1 gpurun_out/bk_ncu.log
