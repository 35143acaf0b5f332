timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
for v in old new old new; do R1_LIB_PATH=$PWD/abtest/$v.so timeout 120 python tools/solve_probe.py C2 C5 --alg hoscf,ihoscf --reps 3 2>&1 | grep rep2 | sed "s/^/$v /" | cut -c1-140; done
