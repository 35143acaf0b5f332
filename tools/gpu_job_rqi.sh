set -x
timeout 600 python tools/solve_probe.py C2 C5 --alg ihoscf,hopm,jacobi_hopm,asvd --reps 2 2>&1 | grep -v "^   it" | tail -20
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/list_rqi_c2.csv python tools/solve_probe.py C2 --alg ihoscf --reps 1 > /dev/null 2>&1
