timeout 60 python tools/solve_probe.py C2 --alg ihoscf --reps 1 2>&1 | grep rep0 || echo TIMEOUT
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
for v in old new old new; do R1_LIB_PATH=$PWD/abtest/$v.so timeout 60 python tools/solve_probe.py C2 C5 --alg ihoscf 2>&1 | grep rep1 | sed "s/^/$v /" | cut -c1-70; done
