"""Randomised parity on fixed seeds (small versions of tools/*_fuzz_probe.py):
random sweeps of orders 2-6 against the oracle restatement, random HOSCF
solves against the compiled reference (lambda and the iteration count),
random Bunch-Kaufman factorisations against the reference's ldlt (pivots
bit-equal), random block operators on the tiled grid Lanczos against numpy."""
import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def test_random_sweeps(gpu_ctx, oracle):
    import paper_2403_01778_b200 as r1
    rng = np.random.default_rng(2024)
    for _ in range(150):
        d = int(rng.integers(2, 7))
        cap = {2: 700, 3: 160, 4: 40, 5: 16, 6: 9}[d]
        dims = tuple(int(rng.integers(1, cap + 1)) for _ in range(d))
        if rng.random() < 0.3:
            dims = tuple(max(1, (k // 8) * 8) for k in dims)
        a = oracle.oracle_random_tensor(dims, int(rng.integers(1 << 30)))
        f = oracle.oracle_random_unit_factors(dims, int(rng.integers(1 << 30)))
        got = r1.build_j(r1.DenseTensor(dims, a), r1.FactorSet(0.0, f)).blocks
        want = oracle.build_j(a, dims, f)
        scale = oracle.build_j_numpy(np.abs(a), dims, [np.abs(u) for u in f])
        assert np.all(np.abs(got - want) <= 1e-13 * scale + 1e-300), dims


def test_fresh_plans_high_order(gpu_ctx, oracle):
    """A NEW sweep plan per shape on small order 4-6 tensors, each swept right
    after its plan metadata went up (the window of the round-2 upload race:
    a fresh plan's segment tables must be on the device before its first box
    kernel, launched as a programmatic dependent, reads them)."""
    import paper_2403_01778_b200 as r1
    rng = np.random.default_rng(4242)
    for _ in range(400):
        d = int(rng.integers(4, 7))
        cap = {4: 40, 5: 12, 6: 8}[d]
        dims = tuple(int(rng.integers(1, cap + 1)) for _ in range(d))
        a = oracle.oracle_random_tensor(dims, int(rng.integers(1 << 30)))
        f = oracle.oracle_random_unit_factors(dims, int(rng.integers(1 << 30)))
        got = r1.build_j(r1.DenseTensor(dims, a), r1.FactorSet(0.0, f)).blocks
        want = oracle.build_j(a, dims, f)
        scale = oracle.build_j_numpy(np.abs(a), dims, [np.abs(u) for u in f])
        assert np.all(np.abs(got - want) <= 1e-13 * scale + 1e-300), dims


def test_random_hoscf_solves(gpu_ctx, oracle, ref):
    import paper_2403_01778_b200 as r1
    rng = np.random.default_rng(77)
    done = 0
    while done < 30:
        d = int(rng.integers(3, 7))
        cap = {3: 60, 4: 20, 5: 10, 6: 7}[d]
        dims = tuple(int(rng.integers(2, cap + 1)) for _ in range(d))
        a = oracle.oracle_random_tensor(dims, int(rng.integers(1 << 30)))
        seed = int(rng.integers(100))
        rep = r1.solve("hoscf", r1.DenseTensor(dims, a), r1.SolveOptions(tol=1e-10, max_iters=300, seed=seed))
        w = ref.solve("hoscf", a, dims, tol=1e-10, max_iters=300, seed=seed)
        assert abs(rep.result.lambda_ - w["lam"]) <= 1e-9 * max(1.0, abs(w["lam"])), dims
        assert abs(rep.iterations - w["iterations"]) <= 1, (dims, seed, rep.iterations, w["iterations"])
        done += 1


def test_random_bunch_kaufman(gpu_ctx, ref):
    from test_bk_gpu import dev_ldlt, ref_d
    rng = np.random.default_rng(99)
    for _ in range(120):
        n = max(1, int(rng.choice([int(rng.integers(1, 130)), 32 * int(rng.integers(1, 12)) + int(rng.integers(-2, 3))])))
        m = rng.standard_normal((n, n))
        s = m + m.T
        kind = int(rng.integers(3))
        if kind == 1:
            np.fill_diagonal(s, 0.0)
        elif kind == 2:
            np.fill_diagonal(s, 1e-3 * rng.standard_normal(n))
        ipiv, diag, sub, sing, cond = dev_ldlt(gpu_ctx, s)
        w, ipr, singr, condr = ref.ldlt(s)
        assert sing == singr and np.array_equal(ipiv, ipr), (n, kind)
        if not sing:
            dr, sr = ref_d(w, ipr)
            sc = np.max(np.abs(s))
            assert np.max(np.abs(diag - dr)) <= 1e-10 * sc and np.max(np.abs(sub - sr)) <= 1e-10 * sc


def test_random_tiled_lanczos(gpu_ctx):
    import paper_2403_01778_b200 as r1
    rng = np.random.default_rng(5)
    for _ in range(25):
        d = int(rng.integers(2, 7))
        while True:
            dims = [int(rng.integers(1, 1400)) if rng.random() < 0.3 else int(rng.integers(1, 300))
                    for _ in range(d)]
            if 1024 < sum(dims) <= 1800:
                break
        dims = tuple(dims)
        nb = sum(dims[m] * dims[k] for m in range(d) for k in range(m + 1, d))
        j = r1.SymBlockMatrix(dims, rng.standard_normal(nb))
        pair, info = r1.eig_blocks(j)
        w, v = np.linalg.eigh(j.dense())
        k = 0 if abs(w[0]) > abs(w[-1]) * (1 + 1e-12) else -1
        vec = v[:, k]
        i = int(np.argmax(np.abs(vec)))
        vec = vec if vec[i] > 0 else -vec
        assert info["converged"] == 1, (dims, info)
        assert abs(pair.value - w[k]) <= 1e-12 * abs(w[k]), dims
        gap = min(abs(abs(w[0]) - abs(w[-1])), abs(w[-1] - w[-2]), abs(w[1] - w[0])) / max(abs(w[0]), abs(w[-1]))
        if gap > 1e-6:
            assert np.max(np.abs(pair.vector - vec)) <= 1e-8, dims
