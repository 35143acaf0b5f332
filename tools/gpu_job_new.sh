set -x
timeout 900 python -m pytest tests/test_experiment_gpu.py tests/test_greedy_io_gpu.py -q -x 2>&1 | tail -25
python -m paper_2403_01778_b200.experiment --generator exp --algos hoscf,ihoscf,hopm,jacobi_hopm,asvd,jacobi_asvd --seeds 3 --tol 1e-8 2>&1 | tail -30
