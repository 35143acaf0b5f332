"""Parity of the device eigen step, RQI step, Eq. 11, KKT and the full
HOSCF / iHOSCF solvers with the compiled reference (oracle/_ref) on seeded
inputs.  Tolerances follow BASELINE.json's north star: sigma within 1e-10
relative, factors within 1e-8 up to sign, iteration count within +-1."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _blocks(oracle, dims, seed):
    a = oracle.oracle_random_tensor(dims, seed)
    f = oracle.oracle_random_unit_factors(dims, seed + 1)
    return a, f, oracle.build_j(a, dims, f)


@pytest.mark.parametrize("dims", [(3, 4), (5, 7), (2, 2, 2), (7, 5, 9), (30, 20, 10),
                                  (6, 5, 4, 3), (4, 3, 5, 2, 3), (40, 30, 20), (100, 100, 100),
                                  (20, 20, 20, 20),
                                  # n = 301 (odd), 1024 (largest single-cluster
                                  # kernel: J rows in L2), 1025 (grid kernel)
                                  (101, 100, 100), (400, 324, 300), (400, 325, 300),
                                  # tiled grid kernel (n > 1024): d = 2, a 2-row mode
                                  # (row chunks of 2), d = 4, odd extents, rows over
                                  # several 256-row chunks
                                  (500, 600), (2, 3, 1100), (800, 200, 20, 10), (257, 513, 301),
                                  (1100, 60, 7)])
def test_eig_blocks_matches_reference(gpu_ctx, oracle, ref, dims):
    import paper_2403_01778_b200 as r1
    a, f, blocks = _blocks(oracle, dims, 31)
    j = r1.SymBlockMatrix(dims, blocks)
    pair, info = r1.eig_blocks(j)
    assert info["converged"] == 1, info
    val, vec = ref.largest_magnitude_eigenpair(ref.block_dense(dims, blocks))
    assert abs(pair.value - val) <= 1e-12 * abs(val), (pair.value, val, info)
    # the pick/sign rules make the vector unique when the eigenvalue is simple
    assert np.max(np.abs(pair.vector - vec)) <= 1e-8, (np.max(np.abs(pair.vector - vec)), info)


def test_eig_symmetric_spectrum_tie_picks_positive(gpu_ctx, oracle, ref):
    """d = 2: J = [[0,A],[A',0]] has the exact +-sigma tie; sym_eig.cpp:214-216 picks +."""
    import paper_2403_01778_b200 as r1
    dims = (5, 7)
    a = oracle.oracle_random_tensor(dims, 10)
    j = r1.SymBlockMatrix(dims, a)
    pair, _ = r1.eig_blocks(j)
    val, vec = ref.largest_magnitude_eigenpair(ref.block_dense(dims, a))
    assert pair.value > 0 and abs(pair.value - val) <= 1e-12 * val
    assert np.max(np.abs(pair.vector - vec)) <= 1e-8


@pytest.mark.parametrize("n", [2, 5, 40, 200])
def test_dense_eigenpair_api(gpu_ctx, oracle, ref, n):
    import paper_2403_01778_b200 as r1
    rng = np.random.default_rng(n)
    m = rng.standard_normal((n, n))
    s = m + m.T
    p = r1.largest_magnitude_eigenpair(s)
    val, vec = ref.largest_magnitude_eigenpair(s)
    assert abs(p.value - val) <= 1e-12 * abs(val)
    assert np.max(np.abs(p.vector - vec)) <= 1e-8
    with pytest.raises(ValueError, match="not symmetric"):
        r1.largest_magnitude_eigenpair(m + 3 * np.eye(n) if n > 1 else np.array([[1.0, 2.0], [0.0, 1.0]]))


def test_rqi_step_matches_reference(gpu_ctx, oracle, ref):
    import paper_2403_01778_b200 as r1
    dims = (7, 5, 9)
    a, f, blocks = _blocks(oracle, dims, 40)
    s = ref.block_dense(dims, blocks)
    x = oracle.stack_factors(f)
    y = r1.rayleigh_quotient_step(s, x)
    yr = ref.rayleigh_quotient_step(s, x)
    assert (y is None) == (yr is None)
    if yr is not None:
        sgn = 1.0 if np.dot(y, yr) > 0 else -1.0
        assert np.max(np.abs(sgn * y - yr)) <= 1e-8
    # 2x2 hand case (test_sym_eig.cpp:191-202): S = diag(2,1), x = (1,1)/sqrt2 -> (1,-1)/sqrt2
    r = 1.0 / np.sqrt(2.0)
    y2 = r1.rayleigh_quotient_step(np.diag([2.0, 1.0]), np.array([r, r]))
    assert y2 is not None
    assert abs(y2[0] - r) <= 1e-12 * r and abs(y2[1] + r) <= 1e-12 * r


def test_eig_kats(gpu_ctx):
    """test_sym_eig.cpp:103-111, 134-141 on the device eigen path."""
    import paper_2403_01778_b200 as r1
    p = r1.largest_magnitude_eigenpair(np.diag([-5.0, 3.0]))
    assert abs(p.value + 5.0) <= 1e-14 and abs(abs(p.vector[0]) - 1.0) <= 1e-14 and p.vector[0] > 0
    p = r1.largest_magnitude_eigenpair(np.array([[0.0, 1.0], [1.0, 0.0]]))
    assert abs(p.value - 1.0) <= 1e-14 and p.value > 0


def test_eq11_and_kkt_match_reference(gpu_ctx, oracle, ref):
    import paper_2403_01778_b200 as r1
    for dims in [(7, 5, 9), (6, 5, 4, 3), (3, 4)]:
        a, f, blocks = _blocks(oracle, dims, 50)
        x = oracle.stack_factors(f)
        j = r1.SymBlockMatrix(dims, blocks)
        got = r1.scf_stopping_value(j, r1.StackedVector(dims, x), 1.3)
        want = ref.scf_stopping_value(dims, blocks, x, 1.3)
        assert abs(got - want) <= 1e-12 * want
        k = r1.kkt_report(r1.DenseTensor(dims, a), r1.FactorSet(0.0, f))
        lam, mx, res = ref.kkt_report(a, dims, f)
        assert abs(k.lambda_ - lam) <= 1e-12 * abs(lam)
        assert abs(k.max_residual - mx) <= 1e-12 * abs(lam)
    # Eq. 11 hand case (test_nepv.cpp:260-276)
    j = r1.build_j(r1.DenseTensor([1, 1], [1.0]), r1.FactorSet(0.0, [[1.0], [1.0]]))
    v = r1.scf_stopping_value(j, r1.StackedVector([1, 1], [1.0, 0.0]), 1.0)
    assert abs(v - 1.0 / (np.sqrt(2.0) + 1.0)) <= 1e-14


SOLVE_CASES = [
    ("hoscf", (4, 5, 6), "rank1", 1e-4, 5),
    ("hoscf", (30, 30, 30), "exp", 1e-4, 0),
    ("ihoscf", (30, 30, 30), "exp", 1e-4, 0),
    ("hoscf", (7, 5, 9), "gauss", 1e-10, 1),
    ("ihoscf", (7, 5, 9), "gauss", 1e-10, 1),
    ("hoscf", (5, 7), "gauss", 1e-10, 1),
    ("hoscf", (10, 10, 10, 10, 10), "tan", 1e-4, 0),
    ("ihoscf", (10, 10, 10, 10, 10), "tan", 1e-4, 0),
    ("hoscf", (6, 5, 4, 3), "gauss", 1e-8, 3),
    ("ihoscf", (20, 20, 20), "c1", 1e-10, 1),
]

# iHOSCF on tensors whose iteration stagnates near the tolerance: the RQI
# accept test |rho_y| > |rho_mid| compares two Rayleigh quotients equal to the
# last ulp there, so the iteration count is sensitive to rounding — in the
# reference itself (test_reference_sensitivity below: 1-ulp input
# perturbations move it over 118-122 and 41-45).  The device path still meets
# the north star's +-1 on the unperturbed inputs; test_chaotic_distribution
# checks it against the reference's own spread.
CHAOTIC = {("ihoscf", (20, 20, 20), "c1"), ("ihoscf", (7, 5, 9), "gauss")}


def _input(oracle, ref, dims, kind):
    if kind == "rank1":
        f = oracle.oracle_random_unit_factors(dims, 3)
        t = np.einsum("i,j,k->ijk", *f) * 7.0
        return t.reshape(-1, order="F")
    if kind in ("exp", "tan"):
        return ref.generate(kind, dims)
    if kind == "c1":
        return oracle.gen_config(1, dims, 1)
    return oracle.oracle_random_tensor(dims, 11)


@pytest.mark.parametrize("alg,dims,kind,tol,seed", SOLVE_CASES)
def test_solver_matches_reference(gpu_ctx, oracle, ref, alg, dims, kind, tol, seed):
    import paper_2403_01778_b200 as r1
    a = _input(oracle, ref, dims, kind)
    want = ref.solve(alg, a, dims, tol=tol, max_iters=500, seed=seed)
    got = r1.solve(alg, r1.DenseTensor(dims, a), r1.SolveOptions(tol=tol, max_iters=500, seed=seed))
    assert got.converged == want["converged"]
    assert abs(got.iterations - want["iterations"]) <= 1, (got.iterations, want["iterations"])
    assert abs(got.result.lambda_ - want["lam"]) <= 1e-10 * abs(want["lam"]), (got.result.lambda_, want["lam"])
    if got.iterations == want["iterations"]:
        for u, v in zip(got.result.factors, want["factors"]):
            assert min(np.max(np.abs(u - v)), np.max(np.abs(u + v))) <= 1e-8
    assert got.result.lambda_ >= 0
    assert len(got.trace) == got.iterations
    assert abs(got.lambda0 - want["lambda0"]) <= 1e-12 * max(1.0, abs(want["lambda0"]))


def test_solver_validation(gpu_ctx):
    import paper_2403_01778_b200 as r1
    a = r1.DenseTensor([3, 3], np.arange(9.0))
    with pytest.raises(ValueError, match="tol must be > 0"):
        r1.hoscf(a, r1.SolveOptions(tol=0.0))
    with pytest.raises(ValueError, match="max_iters"):
        r1.hoscf(a, r1.SolveOptions(max_iters=0))
    with pytest.raises(ValueError, match="unknown solver"):
        r1.solve("nope", a, r1.SolveOptions())
    with pytest.raises(ValueError, match="tol must be > 0"):
        r1.solve("hopm", a, r1.SolveOptions(tol=0.0))


def _perturbed(a, t, rng):
    return a.copy() if t == 0 else a * (1 + rng.choice([-1, 0, 1], size=a.size) * 2.0 ** -52)


@pytest.mark.parametrize("case", sorted(CHAOTIC))
def test_chaotic_distribution(gpu_ctx, oracle, ref, case):
    """Over the input and 11 one-ulp perturbations of it, the device iteration
    counts of a stagnating iHOSCF case stay inside the reference's own range
    widened by its spread, and the medians agree within that spread."""
    import paper_2403_01778_b200 as r1
    alg, dims, kind = case
    a = _input(oracle, ref, dims, kind)
    rng = np.random.default_rng(0)
    ref_its, gpu_its = [], []
    for t in range(12):
        b = _perturbed(a, t, rng)
        ref_its.append(ref.solve(alg, b, dims, tol=1e-10, max_iters=500, seed=1)["iterations"])
        gpu_its.append(r1.solve(alg, r1.DenseTensor(dims, b),
                                r1.SolveOptions(tol=1e-10, max_iters=500, seed=1)).iterations)
    spread = max(ref_its) - min(ref_its)
    assert spread >= 2  # the case is genuinely rounding-sensitive in the reference
    assert min(ref_its) - spread <= min(gpu_its) and max(gpu_its) <= max(ref_its) + spread, (ref_its, gpu_its)
    assert abs(np.median(gpu_its) - np.median(ref_its)) <= spread, (ref_its, gpu_its)


@pytest.mark.parametrize("dims,seed", [((500, 600), 5), ((700, 400, 3), 6)])
def test_tiled_lanczos_long_krylov(gpu_ctx, oracle, dims, seed):
    """The tiled grid Lanczos kernel (n > 1024) from a cold start on operators
    whose extreme eigenvalues are clustered (Gaussian blocks): the Krylov space
    grows past the 32 vectors whose pass-2 dots are held in registers, so the
    memory path for k >= 32 runs; value and vector against numpy's dense
    eigensolver with the reference's pick and sign rules."""
    import paper_2403_01778_b200 as r1
    rng = np.random.default_rng(seed)
    if len(dims) == 2:
        blocks = rng.standard_normal(dims[0] * dims[1])
    else:
        a = rng.standard_normal(int(np.prod(dims)))
        f = [u / np.linalg.norm(u) for u in (rng.standard_normal(k) for k in dims)]
        blocks = r1.build_j(r1.DenseTensor(dims, a), r1.FactorSet(0.0, f)).blocks
    j = r1.SymBlockMatrix(dims, blocks)
    pair, info = r1.eig_blocks(j)
    assert info["converged"] == 1, info
    assert info["steps"] > 32 or info["restarts"] > 0, info
    w, v = np.linalg.eigh(j.dense())
    lo, hi = w[0], w[-1]
    k = 0 if abs(lo) > abs(hi) * (1 + 1e-12) else -1
    want, vec = w[k], v[:, k]
    i = int(np.argmax(np.abs(vec)))
    vec = vec if vec[i] > 0 else -vec
    assert abs(pair.value - want) <= 1e-12 * abs(want), (pair.value, want, info)
    assert np.max(np.abs(pair.vector - vec)) <= 1e-8, (np.max(np.abs(pair.vector - vec)), info)
