set -x
timeout 900 python -m pytest tests/test_bk_gpu.py tests/test_solver_gpu.py -q 2>&1 | tail -5
timeout 300 python tools/bk_probe.py 2>&1 | tail -6
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/list_bk.csv python tools/bk_probe.py 6500 > /dev/null 2>&1
