for G in 1 148; do
R1_EIG_GRID=$G R1_DEBUG_EIG=1 timeout 120 python tools/eig_dense_probe.py 120 129 131 140 2>&1 | grep -E "r1 eig" | awk '{print $3, $6, $7, $8, $9}'
done
timeout 900 python -m pytest tests/test_nepv_props_gpu.py tests/test_solver_gpu.py tests/test_solver_props_gpu.py tests/test_baselines_gpu.py -q 2>&1 | tail -2
