"""Known-answer and property cases of the reference's unit tests that the
other GPU files do not restate (proj/tests/test_nepv.cpp, test_sym_eig.cpp,
test_solvers.cpp), on the device path."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _r1():
    import paper_2403_01778_b200 as r1
    return r1


def test_build_block_of_a_matrix_is_the_matrix(gpu_ctx, oracle):
    """test_nepv.cpp:70-79 (exact)."""
    r1 = _r1()
    a = oracle.oracle_random_tensor((3, 5), 4)
    f = oracle.oracle_random_unit_factors((3, 5), 5)
    b = r1.build_block(r1.DenseTensor((3, 5), a), r1.FactorSet(0.0, f), 0, 1)
    assert np.array_equal(np.asarray(b).reshape(-1, order="F"), a)


def test_build_j_of_a_matrix_is_the_zero_diagonal_embedding(gpu_ctx, oracle):
    """test_nepv.cpp:110-124: scale 1, J = [[0, A], [A', 0]] exactly."""
    r1 = _r1()
    a = oracle.oracle_random_tensor((3, 4), 9)
    f = oracle.oracle_random_unit_factors((3, 4), 10)
    j = r1.build_j(r1.DenseTensor((3, 4), a), r1.FactorSet(0.0, f))
    assert j.scale() == 1.0
    d = j.dense()
    m = a.reshape((3, 4), order="F")
    assert np.array_equal(d[:3, 3:], m) and np.array_equal(d[3:, :3], m.T)
    assert np.all(d[:3, :3] == 0.0)


def test_build_j_reuse_option_matches_direct(gpu_ctx, oracle):
    """test_nepv.cpp:211-225: reuse_intermediates (the device sweep always
    reuses) equals build_j_serial to 1e-12."""
    r1 = _r1()
    dims = (3, 4, 3, 2, 2)
    a = oracle.oracle_random_tensor(dims, 18)
    f = r1.FactorSet(0.0, oracle.oracle_random_unit_factors(dims, 19))
    ref = r1.build_j_serial(r1.DenseTensor(dims, a), f).blocks
    got = r1.build_j(r1.DenseTensor(dims, a), f, r1.BuildOptions(reuse_intermediates=True)).blocks
    assert np.all(np.abs(got - ref) <= 1e-12 * np.maximum(np.abs(ref), 1e-300))


def test_build_j_rejects_a_zero_factor(gpu_ctx, oracle):
    """test_nepv.cpp:227-232: std::runtime_error."""
    r1 = _r1()
    a = oracle.oracle_random_tensor((3, 3, 3), 20)
    f = oracle.oracle_random_unit_factors((3, 3, 3), 21)
    f[2] = np.zeros(3)
    with pytest.raises(RuntimeError):
        r1.build_j(r1.DenseTensor((3, 3, 3), a), r1.FactorSet(0.0, f))


def test_kkt_at_an_exact_singular_pair(gpu_ctx, oracle):
    """test_nepv.cpp:234-241: lambda 6.5 to 1e-12, residual <= 1e-12 * 6.5."""
    r1 = _r1()
    dims = (4, 3, 5)
    f = oracle.oracle_random_unit_factors(dims, 22)
    a = oracle.rank_one_expand(6.5, f, dims)
    k = r1.kkt_report(r1.DenseTensor(dims, a), r1.FactorSet(6.5, f))
    assert abs(k.lambda_ - 6.5) <= 1e-12 * 6.5 and k.max_residual <= 1e-12 * 6.5


def test_kkt_for_the_top_singular_pair_of_a_matrix(gpu_ctx, oracle):
    """test_nepv.cpp:243-258: |lambda| = sigma_1 to 1e-10 and a stationary
    residual; generic unit factors are not stationary (> 1e-3) and
    max_residual is the largest per-mode residual."""
    r1 = _r1()
    a = oracle.oracle_random_tensor((5, 7), 23)
    u, s, vt = np.linalg.svd(a.reshape((5, 7), order="F"))
    k = r1.kkt_report(r1.DenseTensor((5, 7), a), r1.FactorSet(0.0, [u[:, 0], vt[0]]))
    assert abs(abs(k.lambda_) - s[0]) <= 1e-10 * s[0] and k.max_residual <= 1e-10 * s[0]
    g = r1.kkt_report(r1.DenseTensor((5, 7), a), r1.FactorSet(0.0, oracle.oracle_random_unit_factors((5, 7), 24)))
    assert g.max_residual > 1e-3 and g.max_residual == max(g.per_mode_residuals)


def test_exact_plus_minus_tie_resolves_to_positive(gpu_ctx):
    """test_sym_eig.cpp:134-141: S = [[0,1],[1,0]] -> +1."""
    r1 = _r1()
    p = r1.largest_magnitude_eigenpair(np.array([[0.0, 1.0], [1.0, 0.0]]))
    assert abs(p.value - 1.0) <= 1e-14 and p.value > 0.0


def test_rqi_contracts_the_angle_near_a_separated_eigenvector(gpu_ctx):
    """test_sym_eig.cpp:222-252 (same construction, numpy-seeded): spectrum
    0, 0.1, ..., 0.8, 3.0; from the top eigenvector perturbed by 1e-3 one RQI
    step reduces the angle at least 100-fold."""
    r1 = _r1()
    n = 10
    rng = np.random.default_rng(31)
    q, _ = np.linalg.qr(rng.standard_normal((n, n)))
    target = 0.1 * np.arange(n)
    target[-1] = 3.0
    s = (q * target) @ q.T
    s = np.triu(s) + np.triu(s, 1).T
    v = np.linalg.eigh(s)[1][:, -1]
    x = v + 1e-3 * np.random.default_rng(77).standard_normal(n)
    x /= np.linalg.norm(x)
    before = np.arccos(min(1.0, abs(np.dot(x, v))))
    y = r1.rayleigh_quotient_step(s, x)
    assert y is not None
    after = np.arccos(min(1.0, abs(np.dot(y, v))))
    assert after <= before / 100.0, (before, after)


def test_hoscf_quick_statistics_on_the_exp_tensor(gpu_ctx, ref):
    """test_solvers.cpp:90-103: three seeds on the 30^3 exp tensor: converged,
    rho = lambda / ||A||_F within 2% of 0.8207, <= 30 iterations, and the
    report contract (lambda >= 0, unit factors, trace length = iterations)."""
    r1 = _r1()
    a = ref.generate("exp", (30, 30, 30))
    fro = np.linalg.norm(a)
    for seed in range(3):
        rep = r1.hoscf(r1.DenseTensor((30, 30, 30), a), r1.SolveOptions(seed=seed))
        assert rep.converged and rep.iterations <= 30
        assert abs(rep.result.lambda_ / fro - 0.8207) <= 0.02 * 0.8207
        assert rep.result.lambda_ >= 0.0 and len(rep.trace) == rep.iterations
        for u in rep.result.factors:
            assert abs(np.linalg.norm(u) - 1.0) <= 1e-12
