"""The hand-written Bunch-Kaufman LDL^T (csrc/bk.cu) against the reference's
ldlt_factor / ldlt_diag_condition / rayleigh_quotient_step (sym_eig.cpp:233-438):
the same pivot sequence (ipiv, reference encoding), the same D blocks (1e-10
relative), the same condition estimate, singular detection, and the RQI
solution (1e-8 up to sign) — on random symmetric indefinite matrices crossing
several 32-column panels, matrices built to force 2x2 pivots and interchanges,
rank-deficient ones, and shifted block matrices J(u) - rho I near convergence."""
import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def dev_ldlt(ctx, s):
    from paper_2403_01778_b200 import _lib
    n = s.shape[0]
    f = np.asfortranarray(s, dtype=np.float64).reshape(-1, order="F").copy()
    ipiv = np.empty(n, dtype=np.int32)
    diag, sub = np.empty(n), np.empty(n)
    sing, cond = ctypes.c_int(), ctypes.c_double()
    _lib.check(_lib.lib().r1x_ldlt(ctx.handle, n, _lib.dptr(f), ipiv.ctypes.data_as(ctypes.POINTER(ctypes.c_int)),
                                   _lib.dptr(diag), _lib.dptr(sub), ctypes.byref(sing), ctypes.byref(cond)))
    return ipiv, diag, sub, bool(sing.value), cond.value


def ref_d(w, ipiv):
    n = len(ipiv)
    diag = np.array([w[k, k] for k in range(n)])
    sub = np.zeros(n)
    k = 0
    while k < n:
        if ipiv[k] < 0:
            sub[k] = w[k + 1, k]
            k += 2
        else:
            k += 1
    return diag, sub


def sym(rng, n):
    m = rng.standard_normal((n, n))
    return m + m.T


CASES = ["rand1", "rand2", "rand5", "rand33", "rand100", "rand257", "rand1000", "rand2050", "zero_diag",
         "tiny_diag", "rank_def", "blockJ"]  # rand1000 / rand2050: 4- / 9-CTA panel clusters


def make(case, oracle):
    rng = np.random.default_rng(7)
    if case.startswith("rand"):
        return sym(rng, int(case[4:]))
    if case == "zero_diag":  # forces 2x2 pivots everywhere
        s = sym(rng, 70)
        np.fill_diagonal(s, 0.0)
        return s
    if case == "tiny_diag":  # forces 1x1 interchanges
        s = sym(rng, 90)
        np.fill_diagonal(s, 1e-3 * rng.standard_normal(90))
        return s
    if case == "rank_def":
        u = rng.standard_normal((60, 5))
        return u @ np.diag([3, -2, 1, -1, 0.5]) @ u.T
    dims = (20, 30, 25)
    a = oracle.oracle_random_tensor(dims, 40)
    f = oracle.oracle_random_unit_factors(dims, 41)
    d = oracle.dense(dims, oracle.build_j(a, dims, f))
    return d - 0.3 * np.eye(d.shape[0])


@pytest.mark.parametrize("case", CASES)
def test_ldlt_matches_reference(gpu_ctx, oracle, ref, case):
    s = make(case, oracle)
    ipiv, diag, sub, sing, cond = dev_ldlt(gpu_ctx, s)
    w, ipiv_r, sing_r, cond_r = ref.ldlt(s)
    assert sing == sing_r
    if case == "rank_def":
        # after the 5 genuine pivots the trailing matrix is rounding noise: the
        # pivot choices on noise are arbitrary, the verdict (reject) is not
        assert np.array_equal(ipiv[:5], ipiv_r[:5])
        assert not (cond <= 1e14) and not (cond_r <= 1e14)
        return
    assert np.array_equal(ipiv, ipiv_r), (np.nonzero(ipiv != ipiv_r)[0][:5])
    dr, sr = ref_d(w, ipiv_r)
    scale = np.max(np.abs(s))
    assert np.max(np.abs(diag - dr)) <= 1e-10 * scale
    assert np.max(np.abs(sub - sr)) <= 1e-10 * scale
    if np.isfinite(cond_r):
        assert abs(cond - cond_r) <= 1e-8 * cond_r
    else:
        assert not np.isfinite(cond)


@pytest.mark.parametrize("n", [2, 3, 40, 333])
def test_rqi_step_bk_matches_reference(gpu_ctx, ref, n):
    import paper_2403_01778_b200 as r1
    rng = np.random.default_rng(n)
    s = sym(rng, n)
    x = rng.standard_normal(n)
    x /= np.linalg.norm(x)
    y = r1.rayleigh_quotient_step(s, x)
    yr = ref.rayleigh_quotient_step(s, x)
    assert (y is None) == (yr is None)
    if yr is not None:
        sgn = 1.0 if np.dot(y, yr) > 0 else -1.0
        assert np.max(np.abs(sgn * y - yr)) <= 1e-8


def test_rqi_rejects_near_singular_shift(gpu_ctx, ref):
    """x an exact eigenvector: S - rho I is singular to rounding -> condition
    > 1e14 on both attempts -> nullopt, like the reference."""
    import paper_2403_01778_b200 as r1
    rng = np.random.default_rng(3)
    q, _ = np.linalg.qr(rng.standard_normal((50, 50)))
    s = q @ np.diag(np.linspace(-3, 5, 50)) @ q.T
    s = 0.5 * (s + s.T)
    x = q[:, 7].copy()
    assert (r1.rayleigh_quotient_step(s, x) is None) == (ref.rayleigh_quotient_step(s, x) is None)


def test_rqi_large_n_fallback_paths(gpu_ctx):
    """n = 12000: the panel no longer fits in shared memory (global-memory
    panel kernel) and the cluster solve's rows exceed its shared-memory cap
    (cooperative grid solve).  y = normalised (S - rho I)^-1 x, so
    (S - rho I) y must be parallel to x (backward-stable LDL^T: tiny residual)."""
    import paper_2403_01778_b200 as r1
    n = 12000
    rng = np.random.default_rng(12000)
    m = rng.standard_normal((n, n))
    s = m + m.T
    del m
    x = rng.standard_normal(n)
    x /= np.linalg.norm(x)
    y = r1.rayleigh_quotient_step(s, x)
    assert y is not None
    assert abs(np.linalg.norm(y) - 1.0) <= 1e-12
    rho = float(x @ (s @ x))
    r = s @ y - rho * y
    c = float(x @ r)
    assert np.linalg.norm(r - c * x) <= 1e-9 * np.linalg.norm(r)


def test_rqi_deterministic_multi_cta(gpu_ctx):
    """n = 2500 (10-CTA panel cluster and cluster solve, both exchanging
    st.async messages without cluster barriers): repeated RQI steps are
    bit-identical."""
    import paper_2403_01778_b200 as r1
    n = 2500
    rng = np.random.default_rng(2500)
    m = rng.standard_normal((n, n))
    s = m + m.T
    x = rng.standard_normal(n)
    x /= np.linalg.norm(x)
    y0 = r1.rayleigh_quotient_step(s, x)
    assert y0 is not None
    for _ in range(3):
        assert np.array_equal(r1.rayleigh_quotient_step(s, x), y0)
