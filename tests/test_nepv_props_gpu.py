"""NEPv / eigen properties from the reference suite (proj/tests/test_nepv.cpp,
test_sym_eig.cpp), restated against the device sweep, matvec, eigen step and
RQI."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dims", [(4, 5), (3, 4, 2), (2, 3, 2, 3), (2, 2, 3, 2, 2), (30, 20, 10)])
def test_rayleigh_identity(gpu_ctx, oracle, dims):
    """test_nepv.cpp:157-168: x'J(u)x with x = stack(u) is the multilinear form."""
    import paper_2403_01778_b200 as r1
    a = oracle.oracle_random_tensor(dims, 14 + len(dims))
    f = oracle.oracle_random_unit_factors(dims, 15 + len(dims))
    j = r1.build_j(r1.DenseTensor(dims, a), r1.FactorSet(0.0, f))
    x = oracle.stack_factors(f)
    rho = float(np.dot(x, j.matvec(x)))
    want = oracle.multilinear_value(a, dims, f)
    assert abs(rho - want) <= 1e-10 * max(1.0, abs(want))


@pytest.mark.parametrize("dims", [(3, 4, 2), (2, 3, 2, 2)])
def test_spectral_antisymmetry_under_first_block_flip(gpu_ctx, oracle, dims):
    """test_nepv.cpp:170-182: flipping u_0 negates the spectrum of J, so the
    device eigen step returns the negated largest-magnitude value (up to the
    +-tie rule) on J(flip(u))."""
    import paper_2403_01778_b200 as r1
    for trial in range(10):
        a = oracle.oracle_random_tensor(dims, 100 + trial)
        f = oracle.oracle_random_unit_factors(dims, 200 + trial)
        g = [-f[0]] + list(f[1:])
        j1 = r1.build_j(r1.DenseTensor(dims, a), r1.FactorSet(0.0, f))
        j2 = r1.build_j(r1.DenseTensor(dims, a), r1.FactorSet(0.0, g))
        e1 = np.linalg.eigvalsh(j1.dense())
        e2 = np.linalg.eigvalsh(j2.dense())
        assert np.max(np.abs(e2 + e1[::-1])) <= 1e-9
        p1, _ = r1.eig_blocks(j1)
        p2, _ = r1.eig_blocks(j2)
        assert abs(abs(p1.value) - abs(p2.value)) <= 1e-12 * abs(p1.value)


def test_accepted_rqi_steps_do_not_increase_residual(gpu_ctx):
    """test_sym_eig.cpp:254-289: from a perturbed eigenvector an accepted RQI
    step never increases ||S y - rho(y) y||."""
    import paper_2403_01778_b200 as r1
    accepted = 0
    for trial in range(40):
        n = 6 + trial % 7
        rng = np.random.default_rng(9000 + trial)
        m = rng.standard_normal((n, n))
        s = m + m.T
        w, v = np.linalg.eigh(s)
        x = v[:, -1] + (1e-2 if trial % 2 else 1e-4) * rng.standard_normal(n)
        x /= np.linalg.norm(x)
        sb = s @ x
        rb = np.linalg.norm(sb - np.dot(x, sb) * x)
        y = r1.rayleigh_quotient_step(s, x)
        if y is None:
            continue
        accepted += 1
        sa = s @ y
        ra = np.linalg.norm(sa - np.dot(y, sa) * y)
        assert ra <= rb * (1.0 + 1e-12)
    assert accepted > 20


def test_largest_magnitude_value_is_max_of_extremes(gpu_ctx):
    """test_sym_eig.cpp:143-150: |mu| = max(|w_min|, |w_max|) on random
    symmetric matrices, through the dense device eigen path."""
    import paper_2403_01778_b200 as r1
    for trial in range(8):
        n = 10 + 17 * trial
        rng = np.random.default_rng(trial)
        m = rng.standard_normal((n, n))
        s = m + m.T
        p = r1.largest_magnitude_eigenpair(s)
        w = np.linalg.eigvalsh(s)
        assert abs(abs(p.value) - max(abs(w[0]), abs(w[-1]))) <= 1e-11 * max(abs(w[0]), abs(w[-1]))
        assert np.linalg.norm(s @ p.vector - p.value * p.vector) <= 1e-9 * abs(p.value)
