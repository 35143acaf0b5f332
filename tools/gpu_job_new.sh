for v in old new old new; do R1_LIB_PATH=$PWD/abtest/$v.so timeout 300 python tools/solve_probe.py C2 C5 --alg ihoscf 2>&1 | grep rep1 | sed "s/^/$v /"; done
