set -x
for G in "" 1; do
R1_EIG_SMALL_ONE_CTA=$G R1_DEBUG_EIG=1 python tools/solve_probe.py C1 --alg hoscf --reps 1 --max-iters 20 --tol 1e-300 2>&1 | tail -4
R1_EIG_SMALL_ONE_CTA=$G R1_DEBUG_EIG=1 python -m paper_2403_01778_b200.experiment --generator exp --algos hoscf --seeds 1 --tol 1e-8 2>&1 | tail -4
R1_EIG_SMALL_ONE_CTA=$G python tools/solve_probe.py C1 C4 --alg hoscf,ihoscf --reps 2 2>&1 | grep -v "   it"
done
