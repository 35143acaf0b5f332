"""The reference's acceptance criteria (proj/tests/acceptance.cpp:59-470,
expected results proj/test_output.txt:36-48), restated on the device path:
the experiment harness, the solvers and greedy deflation run on the GPU; the
inputs come from the compiled reference's generators and the reference tests'
oracles.  Criterion 11 (OpenMP thread-count invariance and cost profile) has
no device counterpart; determinism is tests/test_solver_props_gpu.py."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _r1():
    import paper_2403_01778_b200 as r1
    return r1


def _exp_stats():
    """acceptance.cpp:106-129: 50 seeds of hoscf / ihoscf / jacobi_hopm on the
    30^3 exp tensor, tol 1e-4, through the experiment harness."""
    r1 = _r1()
    from paper_2403_01778_b200.experiment import ExperimentSpec, run_experiment
    spec = ExperimentSpec(generator="exp", seeds=50, algorithms=["hoscf", "ihoscf", "jacobi_hopm"],
                          opts=r1.SolveOptions(tol=1e-4, max_iters=500, record_kkt=False))
    res = run_experiment(spec)
    fewer = sum(1 for i in range(50) if res.rows[50 + i].iters < res.rows[i].iters)
    return res.summaries, fewer


@pytest.fixture(scope="module")
def exp_stats(gpu_ctx):
    return _exp_stats()


def test_criterion1_matrix_case_vs_svd(gpu_ctx, oracle):
    """acceptance.cpp:59-95: order-2 tensors up to 50 x 80 (shapes from the
    reference's CounterRng(11, 60)): sigma within 1e-8, singular vectors
    within 1e-6 rad."""
    r1 = _r1()
    draws = oracle.rng_u64(11, 60, 60)
    worst_l, worst_a = 0.0, 0.0
    for trial in range(30):
        rows = 5 + int(draws[2 * trial] % np.uint64(46))
        cols = 5 + int(draws[2 * trial + 1] % np.uint64(76))
        a = oracle.oracle_random_tensor((rows, cols), 9000 + trial)
        rep = r1.hoscf(r1.DenseTensor((rows, cols), a), r1.SolveOptions(seed=trial, tol=1e-10))
        assert rep.converged, trial
        u, s, vt = np.linalg.svd(a.reshape((rows, cols), order="F"))
        worst_l = max(worst_l, abs(rep.result.lambda_ - s[0]) / s[0])
        for f, v in ((rep.result.factors[0], u[:, 0]), (rep.result.factors[1], vt[0])):
            worst_a = max(worst_a, float(np.arccos(min(1.0, abs(np.dot(f, v))))))
    assert worst_l <= 1e-8 and worst_a <= 1e-6, (worst_l, worst_a)


def test_criterion2_exp_rho(exp_stats):
    """acceptance.cpp:131-142: mean rho 0.82 +- 0.01 for hoscf and ihoscf."""
    s, _ = exp_stats
    assert abs(s[0].mean_rho - 0.82) <= 0.01 and abs(s[1].mean_rho - 0.82) <= 0.01, (s[0].mean_rho,
                                                                                       s[1].mean_rho)


def test_criterion3_arcsin_rho(gpu_ctx):
    """acceptance.cpp:144-160: arcsin tensor (20^4), 50 seeds: mean rho
    0.66 +- 0.02 for hoscf and ihoscf."""
    r1 = _r1()
    from paper_2403_01778_b200.experiment import ExperimentSpec, run_experiment
    res = run_experiment(ExperimentSpec(generator="arcsin", seeds=50, algorithms=["hoscf", "ihoscf"],
                                        opts=r1.SolveOptions(tol=1e-4, record_kkt=False)))
    for s in res.summaries:
        assert abs(s.mean_rho - 0.66) <= 0.02, (s.algo, s.mean_rho)


def test_criterion4_exp_iteration_counts(exp_stats):
    """acceptance.cpp:162-177: hoscf mean iterations in [9, 15], ihoscf in
    [5, 10] and below hoscf on >= 80% of the seeds, jacobi_hopm in [20, 33]."""
    s, fewer = exp_stats
    assert 9.0 <= s[0].mean_iters <= 15.0, s[0].mean_iters
    assert 5.0 <= s[1].mean_iters <= 10.0, s[1].mean_iters
    assert s[1].mean_iters < s[0].mean_iters and fewer >= 40, fewer
    assert 20.0 <= s[2].mean_iters <= 33.0, s[2].mean_iters


def test_criterion5_high_order_gaussian(gpu_ctx):
    """acceptance.cpp:179-225: order-5 / 6 gaussian 10^d tensors (tensor seed
    42), 20 seeds: hoscf (tol 1e-4) mean lambda within 5% of the fully
    converged hopm reference; at d = 6 jacobi_hopm is unstable (>= 30% not
    converged or a > 20% lambda deficit)."""
    r1 = _r1()
    from paper_2403_01778_b200.experiment import ExperimentSpec, run_experiment
    for d in (5, 6):
        base = dict(generator="gaussian", dims=[10] * d, tensor_seed=42, seeds=20)
        scf = run_experiment(ExperimentSpec(algorithms=["hoscf"], **base,
                                            opts=r1.SolveOptions(tol=1e-4, record_kkt=False)))
        ref = run_experiment(ExperimentSpec(algorithms=["hopm"], **base,
                                            opts=r1.SolveOptions(tol=1e-12, stop_rule="lambda_delta",
                                                                 record_kkt=False)))
        m_scf, m_ref = scf.summaries[0].mean_lambda, ref.summaries[0].mean_lambda
        assert abs(m_scf - m_ref) <= 0.05 * m_ref, (d, m_scf, m_ref)
        if d == 6:
            jac = run_experiment(ExperimentSpec(algorithms=["jacobi_hopm"], **base,
                                                opts=r1.SolveOptions(tol=1e-4, stop_rule="kkt",
                                                                     record_kkt=False)))
            s = jac.summaries[0]
            assert (s.runs - s.converged) * 10 >= 3 * s.runs or s.mean_lambda < 0.8 * m_ref


def test_criterion6_equal_block_norms(gpu_ctx, ref):
    """acceptance.cpp:227-261: 40 seeds on gaussian 9^3, 7^4, 5^5 (tensor
    seed 100 + seed), tol 1e-10: >= 100 converged runs, block-norm spread of
    the final eigenvector <= 1e-6."""
    r1 = _r1()
    converged, worst = 0, 0.0
    for dims in ((9, 9, 9), (7, 7, 7, 7), (5, 5, 5, 5, 5)):
        offs = np.concatenate([[0], np.cumsum(dims)]).astype(int)
        for seed in range(40):
            a = ref.generate("gaussian", dims, 100 + seed)
            rep = r1.hoscf(r1.DenseTensor(dims, a), r1.SolveOptions(seed=seed, tol=1e-10, max_iters=500,
                                                                  record_kkt=False))
            if not rep.converged:
                continue
            converged += 1
            x = rep.final_x.flat()
            norms = [np.linalg.norm(x[offs[k]:offs[k + 1]]) for k in range(len(dims))]
            worst = max(worst, max(norms) - min(norms))
    assert converged >= 100 and worst <= 1e-6, (converged, worst)


def test_criterion7_spectral_antisymmetry(gpu_ctx, oracle):
    """acceptance.cpp:263-281: flipping u_0 negates the spectrum of J(u)
    (50 trials on 4x3x5 / 3x2x4x3), within 1e-9, J from the device sweep."""
    r1 = _r1()
    worst = 0.0
    for trial in range(50):
        dims = (4, 3, 5) if trial % 2 == 0 else (3, 2, 4, 3)
        a = oracle.oracle_random_tensor(dims, 700 + trial)
        f = oracle.oracle_random_unit_factors(dims, 800 + trial)
        g = [-f[0]] + list(f[1:])
        e1 = np.linalg.eigvalsh(r1.build_j(r1.DenseTensor(dims, a), r1.FactorSet(0.0, f)).dense())
        e2 = np.linalg.eigvalsh(r1.build_j(r1.DenseTensor(dims, a), r1.FactorSet(0.0, g)).dense())
        worst = max(worst, float(np.max(np.abs(e2 + e1[::-1]))))
    assert worst <= 1e-9, worst


def test_criterion8_2x2x2_grid_oracle(gpu_ctx, ref):
    """acceptance.cpp:283-324: on 20 gaussian 2x2x2 tensors the best of 20
    hoscf seeds reaches the brute-force grid maximum to within 1e-6."""
    r1 = _r1()
    t1 = np.pi * np.arange(1000) / 1000
    u0, u1 = np.cos(t1)[:, None], np.sin(t1)[:, None]
    v0, v1 = np.cos(t1)[None, :], np.sin(t1)[None, :]
    worst = 1e300
    for t in range(20):
        a = ref.generate("gaussian", (2, 2, 2), 500 + t)
        w0 = a[0] * u0 * v0 + a[1] * u1 * v0 + a[2] * u0 * v1 + a[3] * u1 * v1
        w1 = a[4] * u0 * v0 + a[5] * u1 * v0 + a[6] * u0 * v1 + a[7] * u1 * v1
        grid = float(np.max(np.hypot(w0, w1)))
        best = max(r1.hoscf(r1.DenseTensor((2, 2, 2), a), r1.SolveOptions(seed=s, tol=1e-8, max_iters=200))
                   .result.lambda_ for s in range(20))
        worst = min(worst, best / grid)
    assert worst >= 1.0 - 1e-6, worst


def test_criterion9_stopping_contract(gpu_ctx, ref):
    """acceptance.cpp:326-354: every solver, both stop rules, gaussian 8^3 and
    6^4: a converged run's last stop value is <= tol and its KKT residual
    <= 10 tol ||A||_F; >= 40 converged runs."""
    r1 = _r1()
    runs = 0
    for dims in ((8, 8, 8), (6, 6, 6, 6)):
        for algo in r1.solver_names():
            for seed in range(3):
                for rule in ("kkt", "eq11"):
                    a = ref.generate("gaussian", dims, 900 + seed)
                    o = r1.SolveOptions(seed=seed, tol=1e-6 if seed == 2 else 1e-4, stop_rule=rule)
                    rep = r1.solve(algo, r1.DenseTensor(dims, a), o)
                    if not rep.converged:
                        continue
                    runs += 1
                    assert rep.trace[-1].stop_value <= o.tol, (algo, rule)
                    k = r1.kkt_report(r1.DenseTensor(dims, a), rep.result)
                    assert k.max_residual <= 10.0 * o.tol * np.linalg.norm(a), (algo, rule, k.max_residual)
    assert runs >= 40, runs


def test_criterion10_greedy_pythagorean(gpu_ctx, ref):
    """acceptance.cpp:356-389: greedy rank-5 deflation of gaussian 15^3
    tensors: residual ratios non-increasing and, for a converged term,
    ||R_after||^2 = ||R_before||^2 - lambda^2 to 1e-8."""
    r1 = _r1()
    for t in range(10):
        a = ref.generate("gaussian", (15, 15, 15), 40 + t)
        rep = r1.greedy_rank_r(r1.DenseTensor((15, 15, 15), a), 5, "hoscf",
                               r1.SolveOptions(seed=t, tol=1e-9, max_iters=400, record_kkt=False))
        assert rep.completed, rep.failure
        base, prev = np.linalg.norm(a), 1.0
        for r, ratio in enumerate(rep.residual_ratios):
            assert ratio <= prev + 1e-12
            if rep.solves[r].converged:
                before = (1.0 if r == 0 else rep.residual_ratios[r - 1]) * base
                after = ratio * base
                lam = rep.terms[r].lambda_
                assert abs(after * after - (before * before - lam * lam)) <= 1e-8 * before * before
            prev = ratio


def test_criterion12_geometric_residual_decay(gpu_ctx, ref):
    """acceptance.cpp:437-458: hoscf on the 30^3 exp tensor converges at tol
    1e-11 with Eq. 11 residuals decreasing over the last five iterations."""
    r1 = _r1()
    a = ref.generate("exp", (30, 30, 30))
    rep = r1.hoscf(r1.DenseTensor((30, 30, 30), a), r1.SolveOptions(seed=0, tol=1e-11, max_iters=500,
                                                                    record_kkt=False))
    assert rep.converged and len(rep.trace) >= 6
    last = len(rep.trace) - 1
    rate = max(rep.trace[k].eq11_value / rep.trace[k - 1].eq11_value for k in range(last - 4, last + 1))
    assert rate < 1.0, rate
