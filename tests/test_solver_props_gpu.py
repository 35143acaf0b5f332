"""Properties the reference's solver tests check (proj/tests/test_solvers.cpp),
restated against the device solvers: invariances, known answers, failure
diagnostics, determinism, options honoured."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _r1():
    import paper_2403_01778_b200 as r1
    return r1


def test_mode_permutation_and_scaling_invariance(gpu_ctx, oracle):
    """test_solvers.cpp:105-153: lambda is invariant under a mode permutation
    (the factors permute along) and equivariant under scaling."""
    r1 = _r1()
    dims = (7, 5, 9)
    a = oracle.oracle_random_tensor(dims, 11).reshape(dims, order="F")
    o = r1.SolveOptions(tol=1e-10, seed=1)
    base = r1.hoscf(r1.DenseTensor(dims, a.reshape(-1, order="F")), o)
    perm = (2, 0, 1)
    ap = np.transpose(a, perm)
    pdims = tuple(dims[p] for p in perm)
    rp = r1.hoscf(r1.DenseTensor(pdims, ap.reshape(-1, order="F")), o)
    assert abs(rp.result.lambda_ - base.result.lambda_) <= 1e-8 * base.result.lambda_
    for k, p in enumerate(perm):
        u, v = rp.result.factors[k], base.result.factors[p]
        assert abs(abs(np.dot(u, v)) - 1.0) <= 1e-8
    rs = r1.hoscf(r1.DenseTensor(dims, -3.5 * a.reshape(-1, order="F")), o)
    assert abs(rs.result.lambda_ - 3.5 * base.result.lambda_) <= 1e-8 * 3.5 * base.result.lambda_


def test_converged_eigenvector_blocks_have_equal_norms(gpu_ctx, ref):
    """test_solvers.cpp:155-170: at an NEPv solution every block of the stacked
    eigenvector has norm 1/sqrt(d)."""
    r1 = _r1()
    dims = (30, 30, 30)
    rep = r1.hoscf(r1.DenseTensor(dims, ref.generate("exp", dims)), r1.SolveOptions(tol=1e-10))
    assert rep.converged
    x = rep.final_x.flat()
    offs = np.concatenate([[0], np.cumsum(dims)]).astype(int)
    for k in range(3):
        assert abs(np.linalg.norm(x[offs[k]:offs[k + 1]]) - 1 / np.sqrt(3)) <= 1e-6


def test_rank_one_and_negative_weight(gpu_ctx, oracle):
    """test_solvers.cpp:53-74, 172-204: an exact rank-one tensor is recovered in
    at most two iterations by hoscf and ihoscf; a negative weight is absorbed
    into factor 0 (lambda >= 0)."""
    r1 = _r1()
    dims = (4, 5, 6)
    f = oracle.oracle_random_unit_factors(dims, 3)
    for w in (7.0, -2.5):
        a = (w * np.einsum("i,j,k->ijk", *f)).reshape(-1, order="F")
        for alg in ("hoscf", "ihoscf"):
            rep = r1.solve(alg, r1.DenseTensor(dims, a), r1.SolveOptions(tol=1e-10, seed=5))
            assert rep.converged and rep.iterations <= 2
            assert abs(rep.result.lambda_ - abs(w)) <= 1e-10 * abs(w)
            t = rep.result.lambda_ * np.einsum("i,j,k->ijk", *rep.result.factors)
            assert np.linalg.norm(t.reshape(-1, order="F") - a) <= 1e-8


def test_matrix_is_top_singular_pair(gpu_ctx, oracle):
    """test_solvers.cpp:76-88: on an order-2 tensor HOSCF finds sigma_1 and its
    singular vectors."""
    r1 = _r1()
    dims = (5, 7)
    m = oracle.oracle_random_tensor(dims, 11).reshape(dims, order="F")
    rep = r1.hoscf(r1.DenseTensor(dims, m.reshape(-1, order="F")), r1.SolveOptions(tol=1e-12))
    u, s, vt = np.linalg.svd(m)
    assert abs(rep.result.lambda_ - s[0]) <= 1e-8 * s[0]
    assert abs(abs(np.dot(rep.result.factors[0], u[:, 0])) - 1) <= 1e-8
    assert abs(abs(np.dot(rep.result.factors[1], vt[0])) - 1) <= 1e-8


def test_ihoscf_needs_fewer_iterations_on_exp(gpu_ctx, ref):
    """test_solvers.cpp:184-204 (exp tensor): iHOSCF converges in fewer
    iterations than HOSCF and to the same value; the signed accept rule also
    converges (:230-239)."""
    r1 = _r1()
    dims = (30, 30, 30)
    a = r1.DenseTensor(dims, ref.generate("exp", dims))
    h = r1.hoscf(a, r1.SolveOptions(tol=1e-8))
    i = r1.ihoscf(a, r1.SolveOptions(tol=1e-8))
    s = r1.ihoscf(a, r1.SolveOptions(tol=1e-8, rqi_accept_rule="signed_increase"))
    assert h.converged and i.converged and s.converged
    assert i.iterations < h.iterations
    assert abs(i.result.lambda_ - h.result.lambda_) <= 1e-8 * h.result.lambda_
    assert abs(s.result.lambda_ - h.result.lambda_) <= 1e-8 * h.result.lambda_


def test_kkt_residual_at_convergence(gpu_ctx, oracle):
    """test_solvers.cpp:20-35: the reported KKT residual at a converged
    solution is small relative to ||A||_F."""
    r1 = _r1()
    dims = (6, 5, 4, 3)
    a = oracle.oracle_random_tensor(dims, 7)
    tol = 1e-9
    rep = r1.hoscf(r1.DenseTensor(dims, a), r1.SolveOptions(tol=tol, seed=2))
    assert rep.converged and rep.trace[-1].stop_value <= tol
    k = r1.kkt_report(r1.DenseTensor(dims, a), rep.result)
    assert k.max_residual <= 10.0 * tol * np.linalg.norm(a)


def test_zero_tensor_fails_with_diagnostic(gpu_ctx):
    """test_solvers.cpp:356-362: every solver reports failure after the restart
    on the zero tensor."""
    r1 = _r1()
    z = r1.DenseTensor((3, 4, 5), np.zeros(60))
    for alg in r1.solver_names():
        with pytest.raises(RuntimeError):
            r1.solve(alg, z, r1.SolveOptions())


def test_determinism_and_provided_init(gpu_ctx, ref):
    """test_solvers.cpp:377-402: identical options give bit-identical reports;
    provided factors equal to a converged solution stop after one iteration."""
    r1 = _r1()
    dims = (30, 30, 30)
    a = r1.DenseTensor(dims, ref.generate("exp", dims))
    o = r1.SolveOptions(tol=1e-9, seed=3)
    for alg in ("hoscf", "ihoscf", "hopm", "jacobi_asvd"):
        p, q = r1.solve(alg, a, o), r1.solve(alg, a, o)
        assert p.iterations == q.iterations and p.result.lambda_ == q.result.lambda_
        for u, v in zip(p.result.factors, q.result.factors):
            assert np.array_equal(u, v)
        assert [t.lambda_ for t in p.trace] == [t.lambda_ for t in q.trace]
    base = r1.hoscf(a, r1.SolveOptions(tol=1e-12))
    again = r1.hoscf(a, r1.SolveOptions(tol=1e-9, init="provided", init_factors=base.result.factors))
    assert again.converged and again.iterations == 1


def test_hopm_trace_is_monotone(gpu_ctx, oracle):
    """test_solvers.cpp:262-271: HOPM's lambda never decreases."""
    r1 = _r1()
    dims = (7, 5, 9)
    a = oracle.oracle_random_tensor(dims, 11)
    rep = r1.hopm(r1.DenseTensor(dims, a), r1.SolveOptions(tol=1e-10, seed=1))
    lam = [t.lambda_ for t in rep.trace]
    assert all(lam[i + 1] >= lam[i] - 1e-12 * abs(lam[i]) for i in range(len(lam) - 1))
