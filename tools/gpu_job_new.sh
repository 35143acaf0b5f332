timeout 120 python tools/sweep_probe.py C3 C1 C4 C2 C5 --reps 20 2>&1 | grep median | sed "s/work_elems.*median/median/" | cut -c1-200
timeout 900 python -m pytest tests/test_sweep_gpu.py tests/test_fullsize_gpu.py -q -x 2>&1 | tail -1
