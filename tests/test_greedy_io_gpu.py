"""§8(f) rows 2-3 on the device: greedy rank-R deflation with the residual in
HBM (greedy.cpp:7-35) against the reference's own runs (golden), and .dt1
files straight to / from HBM (tensor_io.cpp:47-100) against a file written by
the reference's write_dt1 and the reference's error messages."""
import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from golden.gen_golden import DT1_DIMS, GREEDY_CASES, solve_input  # noqa: E402

GOLD = np.load(os.path.join(HERE, "golden", "reference_golden.npz"))
REF_DT1 = os.path.join(HERE, "golden", "ref_7x5x9.dt1")


@pytest.mark.parametrize("case", GREEDY_CASES, ids=[c[0] for c in GREEDY_CASES])
def test_greedy_matches_reference(gpu_ctx, case):
    import paper_2403_01778_b200 as r1
    name, solver, kind, dims, r, tol, seed = case
    a = solve_input(kind, dims, seed)
    g = r1.greedy_rank_r(r1.DenseTensor(dims, a), r, solver, r1.SolveOptions(tol=tol, seed=seed))
    meta = GOLD[f"greedy_{name}_meta"]
    assert g.completed == bool(meta[0]) and len(g.terms) == int(meta[1])
    assert g.failure == bytes(GOLD[f"greedy_{name}_failure"]).decode()
    if not g.terms:
        return
    lam = np.array([t.lambda_ for t in g.terms])
    np.testing.assert_allclose(lam, GOLD[f"greedy_{name}_lambdas"], rtol=1e-10)
    np.testing.assert_allclose(g.residual_ratios, GOLD[f"greedy_{name}_ratios"], rtol=1e-9, atol=1e-12)
    fac = GOLD[f"greedy_{name}_factors"]
    o = 0
    for t in g.terms:
        for u in t.factors:
            v = fac[o:o + len(u)]
            o += len(u)
            assert min(np.max(np.abs(u - v)), np.max(np.abs(u + v))) <= 1e-8
    assert [s.algorithm for s in g.solves] == [solver] * len(g.terms)


def test_greedy_validation_and_input_untouched(gpu_ctx, oracle):
    import paper_2403_01778_b200 as r1
    dims = (5, 4, 3)
    a = oracle.oracle_random_tensor(dims, 3)
    t = r1.DeviceTensor.from_host(a, dims)
    with pytest.raises(ValueError, match="rank must be >= 1"):
        r1.greedy_rank_r(t, 0, "hoscf", r1.SolveOptions())
    with pytest.raises(ValueError, match="zero input tensor"):
        r1.greedy_rank_r(r1.DenseTensor(dims, np.zeros(60)), 1, "hoscf", r1.SolveOptions())
    g = r1.greedy_rank_r(t, 2, "hoscf", r1.SolveOptions(tol=1e-8))
    assert g.completed and np.array_equal(t.to_host(), a)
    # the residual ratios are the norms of A - sum of the terms
    res = a.copy()
    for term in g.terms:
        res -= oracle.rank_one_expand(term.lambda_, term.factors, dims)
    assert abs(np.linalg.norm(res) / np.linalg.norm(a) - g.residual_ratios[-1]) <= 1e-12


def test_rank_one_subtract_matches_expand(gpu_ctx, oracle):
    import ctypes

    import paper_2403_01778_b200 as r1
    from paper_2403_01778_b200 import _lib
    dims = (33, 7, 5, 3)
    a = oracle.oracle_random_tensor(dims, 8)
    f = oracle.oracle_random_unit_factors(dims, 9)
    t = r1.DeviceTensor.from_host(a, dims)
    nrm = ctypes.c_double()
    flat = np.concatenate(f)
    _lib.check(_lib.lib().r1_rank_one_subtract(gpu_ctx.handle, t.handle, 1.75, _lib.dptr(flat),
                                               ctypes.byref(nrm)))
    want = a - oracle.rank_one_expand(1.75, f, dims)
    got = t.to_host()
    assert np.max(np.abs(got - want)) <= 1e-15 * np.max(np.abs(a))
    assert abs(nrm.value - np.linalg.norm(want)) <= 1e-13 * np.linalg.norm(want)


def test_dt1_roundtrip_with_reference_file(gpu_ctx, oracle, tmp_path):
    import paper_2403_01778_b200 as r1
    t = r1.read_dt1(REF_DT1)
    assert t.dims == DT1_DIMS
    assert np.array_equal(t.to_host(), oracle.oracle_random_tensor(DT1_DIMS, 21))
    out = tmp_path / "dev.dt1"
    r1.write_dt1(out, t)
    assert out.read_bytes() == open(REF_DT1, "rb").read()  # byte-identical to the reference's writer
    # a larger tensor crosses several 64 MB staging chunks
    dims = (1000, 100, 181)
    big = r1.DeviceTensor.from_host(np.arange(np.prod(dims), dtype=np.float64), dims)
    p = tmp_path / "big.dt1"
    big.write_dt1(p)
    assert os.path.getsize(p) == 7 + 8 * 3 + 8 * int(np.prod(dims))
    back = r1.read_dt1(p)
    assert back.dims == dims and np.array_equal(back.to_host(), np.arange(np.prod(dims), dtype=np.float64))
    # solving a file-loaded tensor equals solving the host tensor
    s1 = r1.hoscf(r1.read_dt1(REF_DT1), r1.SolveOptions(tol=1e-10, seed=1))
    s2 = r1.hoscf(r1.DenseTensor(DT1_DIMS, oracle.oracle_random_tensor(DT1_DIMS, 21)),
                  r1.SolveOptions(tol=1e-10, seed=1))
    assert s1.result.lambda_ == s2.result.lambda_


def test_dt1_errors_match_reference(gpu_ctx, oracle, tmp_path):
    import paper_2403_01778_b200 as r1
    raw = open(REF_DT1, "rb").read()
    cases = [(b"XTEN1\0" + raw[6:], "bad magic"), (raw[:6] + bytes([1]) + raw[7:], "order must be >= 2"),
             (raw[:-8], "truncated payload"), (raw + b"\0", "trailing bytes"),
             (raw[:7] + (0).to_bytes(8, "little") + raw[15:], "invalid dimension"),
             (raw[:7] + (2 ** 40).to_bytes(8, "little") + (2 ** 40).to_bytes(8, "little") + raw[23:],
              "size overflow")]
    for i, (blob, msg) in enumerate(cases):
        p = tmp_path / f"bad{i}.dt1"
        p.write_bytes(blob)
        with pytest.raises(RuntimeError) as e:
            r1.read_dt1(p)
        assert msg in str(e.value)
        with pytest.raises(RuntimeError) as eo:
            oracle.read_dt1(p)
        assert str(e.value) == str(eo.value)
    with pytest.raises(RuntimeError, match="cannot open"):
        r1.read_dt1(tmp_path / "missing.dt1")
