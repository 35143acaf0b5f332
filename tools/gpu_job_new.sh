for g in 16 12 8 6; do R1_BK_G=$g timeout 300 python tools/solve_probe.py C2 C5 --alg ihoscf 2>&1 | grep rep1 | sed "s/^/G=$g /" | cut -c1-60; done
