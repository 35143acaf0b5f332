"""The reference's sweep baselines on the device (solvers.cpp:299-447: hopm,
jacobi_hopm, asvd, jacobi_asvd) against the reference's own runs (golden
fixtures made by tests/golden/gen_golden.py from the compiled reference):
sigma within 1e-10 relative, factors within 1e-8 up to sign, iterations within
+-1, the per-iteration lambda trace within 1e-9, all three stop rules and the
disjoint-pairs ASVD variant."""
import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from golden.gen_golden import BASELINE_SOLVES, solve_input  # noqa: E402

GOLD = np.load(os.path.join(HERE, "golden", "reference_golden.npz"))
RULES = ["kkt", "eq11", "lambda_delta"]


@pytest.mark.parametrize("case", BASELINE_SOLVES, ids=[c[0] for c in BASELINE_SOLVES])
def test_baseline_matches_reference(gpu_ctx, case):
    import paper_2403_01778_b200 as r1
    name, alg, kind, dims, tol, iters, seed, rule, disjoint = case
    a = solve_input(kind, dims, seed)
    got = r1.solve(alg, r1.DenseTensor(dims, a),
                   r1.SolveOptions(tol=tol, max_iters=iters, seed=seed, stop_rule=RULES[rule],
                                   asvd_disjoint_pairs=disjoint))
    meta = GOLD[f"solve_{name}_meta"]
    lam_ref, conv_ref, it_ref = meta[0], bool(meta[1]), int(meta[2])
    assert got.converged == conv_ref
    assert abs(got.iterations - it_ref) <= 1, (got.iterations, it_ref)
    assert abs(got.result.lambda_ - lam_ref) <= 1e-10 * abs(lam_ref), (got.result.lambda_, lam_ref)
    assert abs(got.lambda0 - meta[3]) <= 1e-12 * max(1.0, abs(meta[3]))
    assert got.result.lambda_ >= 0 and len(got.trace) == got.iterations
    assert got.final_x is None
    lt = GOLD[f"solve_{name}_lambda_trace"]
    k = min(len(lt), len(got.trace))
    trace = np.array([t.lambda_ for t in got.trace[:k]])
    assert np.max(np.abs(trace - lt[:k])) <= 1e-9 * np.max(np.abs(lt))
    if got.iterations == it_ref:
        fac = GOLD[f"solve_{name}_factors"]
        o = 0
        for u in got.result.factors:
            v = fac[o:o + len(u)]
            o += len(u)
            assert min(np.max(np.abs(u - v)), np.max(np.abs(u + v))) <= 1e-8
    # one pass over A per sweep: Jacobi forms cost one sweep per iteration
    if alg in ("jacobi_hopm", "jacobi_asvd"):
        assert got.total_sweeps == got.iterations + 1
    if alg == "hopm":
        assert got.total_sweeps == 1 + len(dims) * got.iterations


def test_baseline_kats(gpu_ctx, oracle):
    """test_solvers.cpp-style known answers: a rank-one tensor 7 u o v o w is
    recovered by every baseline in one or two iterations."""
    import paper_2403_01778_b200 as r1
    dims = (4, 5, 6)
    f = oracle.oracle_random_unit_factors(dims, 3)
    a = (np.einsum("i,j,k->ijk", *f) * 7.0).reshape(-1, order="F")
    for alg in ("hopm", "jacobi_hopm", "asvd", "jacobi_asvd"):
        rep = r1.solve(alg, r1.DenseTensor(dims, a), r1.SolveOptions(tol=1e-10, seed=5))
        assert rep.converged and rep.iterations <= 2, (alg, rep.iterations)
        assert abs(rep.result.lambda_ - 7.0) <= 1e-12 * 7.0
        for u, v in zip(rep.result.factors, f):
            assert min(np.max(np.abs(u - v)), np.max(np.abs(u + v))) <= 1e-10
