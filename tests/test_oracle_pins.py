"""Pins the CPU oracle (oracle/rank1_oracle.{c,py}) to the reference:
  * against the golden fixtures produced by the compiled reference
    (tests/golden/reference_golden.npz, tests/golden/gen_golden.py), always;
  * against the live compiled reference (oracle/_ref) when it is built;
  * against the reference's own known-answer tests (test_nepv.cpp,
    test_sym_eig.cpp, test_solvers.cpp).
No GPU: these run in the CPU suite."""
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = np.load(os.path.join(HERE, "golden", "reference_golden.npz"))

from golden.gen_golden import (BASELINE_SOLVES, DT1_DIMS, GREEDY_CASES, SOLVES, SWEEP_SHAPES,  # noqa: E402
                               solve_input)


def tag(dims):
    return "x".join(map(str, dims))


# --------------------------------------------------------------- RNG pins --

@pytest.mark.parametrize("seed,stream", [(0, 1), (5, 2), (123, 77), (2, 3)])
def test_counter_rng_bit_exact(oracle, seed, stream):
    assert np.array_equal(oracle.rng_u64(seed, stream, 64), GOLD[f"rng_u64_{seed}_{stream}"].view(np.uint64))
    assert np.array_equal(oracle.rng_units(seed, stream, 64), GOLD[f"rng_unit_{seed}_{stream}"])
    assert np.array_equal(oracle.rng_gaussians(seed, stream, 65), GOLD[f"rng_gauss_{seed}_{stream}"])


def test_gen_gaussian_bit_exact(oracle):
    assert np.array_equal(oracle.gen_gaussian((7, 5, 9), 3), GOLD["gen_gaussian_7_5_9_s3"])


# ------------------------------------------------------------- sweep pins --

@pytest.mark.parametrize("i,dims", list(enumerate(SWEEP_SHAPES)))
def test_build_j_bit_exact_vs_reference(oracle, i, dims):
    """The oracle's TTV chains reproduce build_j_serial bit for bit."""
    a = oracle.oracle_random_tensor(dims, 11 + i)
    f = oracle.oracle_random_unit_factors(dims, 12 + i)
    assert np.array_equal(oracle.build_j(a, dims, f), GOLD[f"blocks_{tag(dims)}"])


@pytest.mark.parametrize("i,dims", list(enumerate(SWEEP_SHAPES)))
def test_block_operators_vs_reference(oracle, i, dims):
    a = oracle.oracle_random_tensor(dims, 11 + i)
    f = oracle.oracle_random_unit_factors(dims, 12 + i)
    blocks = GOLD[f"blocks_{tag(dims)}"]
    x = oracle.stack_factors(f)
    np.testing.assert_allclose(oracle.matvec(dims, blocks, x), GOLD[f"matvec_{tag(dims)}"],
                               rtol=1e-12, atol=1e-14)
    assert abs(oracle.frobenius(dims, blocks) - GOLD[f"fro_{tag(dims)}"][0]) <= 1e-13 * GOLD[f"fro_{tag(dims)}"][0]
    e = GOLD[f"eq11_{tag(dims)}"][0]
    assert abs(oracle.scf_stopping_value(dims, blocks, x, 1.3) - e) <= 1e-12 * e
    lam, mx, res = oracle.kkt_from_blocks(dims, blocks, f)
    k = GOLD[f"kkt_{tag(dims)}"]
    assert abs(lam - k[0]) <= 1e-12 * abs(k[0])
    np.testing.assert_allclose(res, k[2:], rtol=1e-9, atol=1e-13 * abs(k[0]))


@pytest.mark.parametrize("i,dims", [(i, d) for i, d in enumerate(SWEEP_SHAPES) if sum(d) <= 400])
def test_eigenpair_and_rqi_vs_reference(oracle, i, dims):
    blocks = GOLD[f"blocks_{tag(dims)}"]
    s = oracle.dense(dims, blocks)
    val, vec = oracle.largest_magnitude_eigenpair(s)
    g = GOLD[f"eig_{tag(dims)}"]
    assert abs(val - g[0]) <= 1e-12 * abs(g[0])
    assert np.max(np.abs(vec - g[1:])) <= 1e-8
    f = oracle.oracle_random_unit_factors(dims, 12 + i)
    y = oracle.rqi_step(s, oracle.stack_factors(f))
    gy = GOLD[f"rqi_{tag(dims)}"]
    assert (y is None) == (gy.size == 0)
    if y is not None:
        assert np.max(np.abs(y - gy)) <= 1e-9 * max(1.0, np.max(np.abs(gy)))


@pytest.mark.parametrize("n", [5, 17, 40])
def test_bunch_kaufman_bit_exact(oracle, n):
    s = GOLD[f"ldlt_in_{n}"]
    w, ipiv, sing, cond = oracle.ldlt(s)
    assert np.array_equal(w, GOLD[f"ldlt_w_{n}"].reshape(-1, order="F"))
    assert np.array_equal(ipiv.astype(np.int64), GOLD[f"ldlt_ipiv_{n}"])
    assert cond == GOLD[f"ldlt_cond_{n}"][0] and sing == bool(GOLD[f"ldlt_cond_{n}"][1])


# ------------------------------------------------------------ solver pins --

@pytest.mark.parametrize("case", SOLVES, ids=[c[0] for c in SOLVES])
def test_oracle_solvers_vs_reference(oracle, case):
    name, alg, kind, dims, tol, iters, seed = case
    if kind in ("exp", "tan"):
        pytest.importorskip("oracle.ref")
        from oracle import ref
        if not ref.available():
            pytest.skip("exp/tan generators come from the compiled reference")
    a = solve_input(kind, dims, seed)
    fn = oracle.hoscf if alg == "hoscf" else oracle.ihoscf
    rep = fn(a, dims, oracle.Options(tol=tol, max_iters=iters, seed=seed))
    meta = GOLD[f"solve_{name}_meta"]
    lam_ref, conv_ref, it_ref = meta[0], bool(meta[1]), int(meta[2])
    assert rep.converged == conv_ref
    chaotic = alg == "ihoscf" and not conv_ref
    assert abs(rep.iterations - it_ref) <= (3 if chaotic else 1)
    assert abs(rep.lam - lam_ref) <= 1e-10 * abs(lam_ref)
    assert abs(rep.lambda0 - meta[3]) <= 1e-12 * max(1.0, abs(meta[3]))
    if rep.iterations == it_ref:
        fac = GOLD[f"solve_{name}_factors"]
        o = 0
        for u in rep.factors:
            v = fac[o:o + len(u)]
            o += len(u)
            assert min(np.max(np.abs(u - v)), np.max(np.abs(u + v))) <= 1e-8


@pytest.mark.parametrize("case", BASELINE_SOLVES, ids=[c[0] for c in BASELINE_SOLVES])
def test_oracle_baselines_vs_reference(oracle, case):
    """The numpy restatement of run_power_sweep / run_asvd (solvers.cpp:299-447)
    against the reference's own runs (golden): sigma 1e-10, factors 1e-8 up to
    sign, iterations +-1, per-iteration lambda trace 1e-9."""
    name, alg, kind, dims, tol, iters, seed, rule, disjoint = case
    a = solve_input(kind, dims, seed)
    rep = getattr(oracle, alg)(a, dims, oracle.Options(
        tol=tol, max_iters=iters, seed=seed, stop_rule=["kkt", "eq11", "lambda_delta"][rule],
        asvd_disjoint_pairs=disjoint))
    meta = GOLD[f"solve_{name}_meta"]
    lam_ref, conv_ref, it_ref = meta[0], bool(meta[1]), int(meta[2])
    assert rep.converged == conv_ref
    assert abs(rep.iterations - it_ref) <= 1, (rep.iterations, it_ref)
    assert abs(rep.lam - lam_ref) <= 1e-10 * abs(lam_ref)
    assert abs(rep.lambda0 - meta[3]) <= 1e-12 * max(1.0, abs(meta[3]))
    lt = GOLD[f"solve_{name}_lambda_trace"]
    k = min(len(lt), len(rep.trace))
    got = np.array([t["lambda"] for t in rep.trace[:k]])
    assert np.max(np.abs(got - lt[:k])) <= 1e-9 * np.max(np.abs(lt))
    if rep.iterations == it_ref:
        fac = GOLD[f"solve_{name}_factors"]
        o = 0
        for u in rep.factors:
            v = fac[o:o + len(u)]
            o += len(u)
            assert min(np.max(np.abs(u - v)), np.max(np.abs(u + v))) <= 1e-8


@pytest.mark.parametrize("case", GREEDY_CASES, ids=[c[0] for c in GREEDY_CASES])
def test_oracle_greedy_vs_reference(oracle, case):
    """greedy_rank_r (greedy.cpp:7-35) restated on the oracle solvers."""
    name, solver, kind, dims, r, tol, seed = case
    a = solve_input(kind, dims, seed)
    g = oracle.greedy_rank_r(a, dims, r, solver, oracle.Options(tol=tol, seed=seed))
    meta = GOLD[f"greedy_{name}_meta"]
    assert g["completed"] == bool(meta[0]) and len(g["terms"]) == int(meta[1])
    assert g["failure"] == bytes(GOLD[f"greedy_{name}_failure"]).decode()
    if g["terms"]:
        np.testing.assert_allclose(g["lambdas"], GOLD[f"greedy_{name}_lambdas"], rtol=1e-10)
        np.testing.assert_allclose(g["ratios"], GOLD[f"greedy_{name}_ratios"], rtol=1e-9, atol=1e-12)


def test_oracle_rank_one_expand_kat(oracle):
    """rank_one_expand: out[i0 + I0 i1 + ...] = ((lambda u0[i0]) u1[i1]) ..."""
    dims = (3, 2, 4)
    f = oracle.oracle_random_unit_factors(dims, 7)
    e = oracle.rank_one_expand(2.5, f, dims)
    want = 2.5 * np.einsum("i,j,k->ijk", *f).reshape(-1, order="F")
    np.testing.assert_allclose(e, want, rtol=1e-15)


def test_oracle_dt1_vs_reference_file(oracle, tmp_path):
    """tests/golden/ref_7x5x9.dt1 was written by the reference's write_dt1."""
    path = os.path.join(HERE, "golden", "ref_7x5x9.dt1")
    a, dims = oracle.read_dt1(path)
    assert dims == list(DT1_DIMS)
    assert np.array_equal(a, oracle.oracle_random_tensor(DT1_DIMS, 21))
    out = tmp_path / "o.dt1"
    oracle.write_dt1(out, a, dims)
    assert out.read_bytes() == open(path, "rb").read()
    bad = tmp_path / "bad.dt1"
    raw = open(path, "rb").read()
    for blob, msg in [(b"XTEN1\0" + raw[6:], "bad magic"), (raw[:6] + bytes([1]) + raw[7:], "order must be"),
                      (raw[:-8], "truncated payload"), (raw + b"\0", "trailing bytes"),
                      (raw[:7] + (0).to_bytes(8, "little") + raw[15:], "invalid dimension")]:
        bad.write_bytes(blob)
        with pytest.raises(RuntimeError, match=msg):
            oracle.read_dt1(bad)


# -------------------------------------------------- reference KATs (tests/) --

def test_kat_all_ones_blocks(oracle):
    """test_nepv.cpp:126-137."""
    s = 1.0 / np.sqrt(2.0)
    b = oracle.build_j(np.ones(8), (2, 2, 2), [np.array([s, s])] * 3)
    np.testing.assert_allclose(b, np.sqrt(2.0), rtol=1e-12)


def test_kat_rank_one_block(oracle):
    """test_nepv.cpp:81-89."""
    dims = (3, 4, 5)
    f = oracle.oracle_random_unit_factors(dims, 6)
    a = np.einsum("i,j,k->ijk", *f).reshape(-1, order="F")
    b = oracle.get_block(oracle.build_j(a, dims, f), dims, 0, 1)
    np.testing.assert_allclose(b, np.outer(f[0], f[1]), rtol=1e-12, atol=1e-15)


def test_kat_matrix_embedding(oracle):
    """test_nepv.cpp:110-124: d = 2 gives J = [[0, A], [A', 0]] with scale 1."""
    dims = (3, 4)
    a = oracle.oracle_random_tensor(dims, 9)
    d = oracle.dense(dims, oracle.build_j(a, dims, oracle.oracle_random_unit_factors(dims, 10)))
    m = a.reshape(dims, order="F")
    assert np.array_equal(d[:3, 3:], m) and np.array_equal(d[3:, :3], m.T)
    assert not d[:3, :3].any()


def test_kat_eq11_hand_case(oracle):
    """test_nepv.cpp:260-276."""
    v = oracle.scf_stopping_value((1, 1), np.array([1.0]), np.array([1.0, 0.0]), 1.0)
    assert abs(v - 1.0 / (np.sqrt(2.0) + 1.0)) <= 1e-14
    assert abs(oracle.scf_stopping_value((1, 1), np.array([1.0]), np.array([-1.0, 0.0]), 1.0) - v) <= 1e-14
    assert oracle.scf_stopping_value((1, 1), np.array([1.0]), np.array([np.sqrt(.5), np.sqrt(.5)]), 1.0) <= 1e-14


def test_kat_eigen_tie_and_sign(oracle):
    """test_sym_eig.cpp:103-111 (magnitude beats sign, canonical sign) and
    :134-141 (exact +-mu tie resolves to +)."""
    val, vec = oracle.largest_magnitude_eigenpair(np.diag([-5.0, 3.0]))
    assert val == -5.0 and abs(vec[0]) == 1.0 and vec[0] > 0
    val, vec = oracle.largest_magnitude_eigenpair(np.array([[0.0, 1.0], [1.0, 0.0]]))
    assert abs(val - 1.0) <= 1e-14 and val > 0


def test_kat_rqi_2x2(oracle):
    """test_sym_eig.cpp:191-202: S = diag(2, 1), x = (1,1)/sqrt2, rho = 1.5 ->
    y = (1,-1)/sqrt2."""
    r = 1.0 / np.sqrt(2.0)
    y = oracle.rqi_step(np.diag([2.0, 1.0]), np.array([r, r]))
    assert y is not None
    assert abs(y[0] - r) <= 1e-12 * r and abs(y[1] + r) <= 1e-12 * r


def test_kat_matrix_case_is_svd(oracle):
    """test_solvers.cpp:76-88: on a matrix HOSCF gives the top singular pair."""
    dims = (5, 7)
    a = oracle.oracle_random_tensor(dims, 10)
    rep = oracle.hoscf(a, dims, oracle.Options(tol=1e-10, seed=1))
    s = np.linalg.svd(a.reshape(dims, order="F"), compute_uv=False)
    assert rep.converged and abs(rep.lam - s[0]) <= 1e-8 * s[0]


# --------------------------------------------- live reference (if built) --

def test_live_reference_sweep_bit_exact(oracle, ref):
    for seed, dims in enumerate([(9, 8, 7), (5, 4, 3, 2), (11, 3, 2, 4, 2)]):
        a = oracle.oracle_random_tensor(dims, 100 + seed)
        f = oracle.oracle_random_unit_factors(dims, 200 + seed)
        assert np.array_equal(oracle.build_j(a, dims, f), ref.build_j(a, dims, f))


def test_live_reference_config_generators(oracle, ref):
    """Config 1 = the reference's gen_gaussian, bit for bit."""
    dims = (12, 10, 8)
    assert np.array_equal(oracle.gen_config(1, dims, 1), ref.gen_gaussian(dims, 1))
