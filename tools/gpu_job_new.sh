timeout 60 python tools/c1_probe.py C1 2>&1 | tail -1
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
for v in old new old new; do R1_LIB_PATH=$PWD/abtest/$v.so timeout 60 python tools/c1_probe.py C1 2>&1 | tail -1 | sed "s/^/$v /"; R1_LIB_PATH=$PWD/abtest/$v.so timeout 120 python tools/solve_probe.py C3 C4 --alg hoscf --reps 2 2>&1 | grep rep1 | sed "s/^/$v /" | cut -c1-140; done
