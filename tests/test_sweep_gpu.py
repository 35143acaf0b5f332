"""Parity of the fused device sweep (rank1::build_j replacement) with the
oracle restatement, which is itself pinned bit-exact to the compiled reference
(tests/test_oracle_pins.py).  Tolerance: blocks agree entrywise within
1e-12 * (sum_i |A_i| prod |u_k| bound), i.e. a relative accuracy far tighter
than the north-star's 1e-10 sigma tolerance."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SHAPES = [
    (3, 4), (5, 7), (2, 2, 2), (7, 5, 9), (30, 20, 10), (100, 100, 100), (129, 65, 33),
    (1, 1, 1), (1, 7, 3), (300, 2, 5), (3, 300, 5), (257, 130, 17), (6, 5, 4, 3),
    (4, 3, 5, 2, 3), (2, 3, 4, 5, 6, 2), (20, 20, 20, 20), (10, 10, 10, 10, 10), (65, 64, 3, 3),
    # merged alignment classes (K = 128 / gcd(8 I0, 128) columns per merged
    # column): one tile holding 4 classes, tiles straddling a class boundary,
    # K = 2 and 4 at several row-tile counts, recursion levels with K > 1
    (20, 8, 5), (200, 10, 7), (500, 8, 3), (60, 60, 9), (1000, 4, 3), (60, 8, 5, 3),
    (40, 12, 6, 2), (100, 4, 2, 2, 2),
    # small single-tile faces: KO o-panels per box (KO = 2 and 4)
    (30, 20, 6), (64, 60, 12), (8, 6, 4, 2, 3),
    # 128 < I0 <= 256 unmerged: one 256-row x 30-column tile per column strip
    # (8 rows x 2 columns per lane), ragged last column tile, recursion levels
    (200, 200, 7), (130, 61, 5), (256, 31, 4), (200, 64, 6, 5), (250, 33, 2, 2, 2),
    # the same I0 range merged (K = 2 / 4: wide enough faces), 128-row tiles
    # straddling the class boundary
    (200, 500, 3), (136, 480, 4), (132, 1000, 2),
    # extreme aspect ratios: a long fastest mode, a tiny face with a long
    # outer mode, unit modes
    (100000, 3, 2), (2, 2, 50000), (1, 1, 1, 1, 1000), (5000, 1, 7), (1, 4000, 3),
]


def _bound(o, a, dims, f):
    """Entrywise error scale: the same contraction on |A| and |u|."""
    return o.build_j_numpy(np.abs(a), dims, [np.abs(u) for u in f])


@pytest.mark.parametrize("dims", SHAPES)
def test_build_j_matches_oracle(gpu_ctx, oracle, dims):
    import paper_2403_01778_b200 as r1
    a = oracle.oracle_random_tensor(dims, 11 + len(dims))
    f = oracle.oracle_random_unit_factors(dims, 12 + len(dims))
    want = oracle.build_j(a, dims, f)
    got = r1.build_j(r1.DenseTensor(dims, a), r1.FactorSet(0.0, f)).blocks
    scale = _bound(oracle, a, dims, f)
    err = np.abs(got - want)
    assert np.all(err <= 1e-13 * scale + 1e-300), (dims, float(np.max(err / (scale + 1e-300))))


def test_build_j_all_ones_kat(gpu_ctx):
    """test_nepv.cpp:126-137: every block entry of the all-ones 2x2x2 tensor with
    factors (1/sqrt2, 1/sqrt2) is sqrt(2); scale 0.5."""
    import paper_2403_01778_b200 as r1
    s = 1.0 / np.sqrt(2.0)
    j = r1.build_j(r1.DenseTensor([2, 2, 2], np.ones(8)), r1.FactorSet(0.0, [[s, s]] * 3))
    assert j.scale() == 0.5
    np.testing.assert_allclose(j.blocks, np.sqrt(2.0), rtol=1e-12)


def test_build_j_rank_one_kat(gpu_ctx, oracle):
    """test_nepv.cpp:81-89: rank-one tensor with its own factors -> B(0,1) = u0 u1'."""
    import paper_2403_01778_b200 as r1
    dims = (3, 4, 5)
    f = oracle.oracle_random_unit_factors(dims, 6)
    a = np.einsum("i,j,k->ijk", *f).reshape(-1, order="F")
    b = r1.build_block(r1.DenseTensor(dims, a), r1.FactorSet(1.0, f), 0, 1)
    np.testing.assert_allclose(b, np.outer(f[0], f[1]), rtol=1e-12, atol=1e-15)


def test_build_j_deterministic(gpu_ctx, oracle):
    """Fixed-order reductions: identical inputs give identical bits."""
    import paper_2403_01778_b200 as r1
    dims = (129, 130, 40)
    a = oracle.oracle_random_tensor(dims, 5)
    f = oracle.oracle_random_unit_factors(dims, 6)
    t = r1.DenseTensor(dims, a)
    b1 = r1.build_j(t, r1.FactorSet(0.0, f)).blocks
    b2 = r1.build_j(t, r1.FactorSet(0.0, f)).blocks
    assert np.array_equal(b1, b2)


@pytest.mark.parametrize("dims", [(200, 200, 300), (1000, 64, 50), (60, 60, 60, 60)])
def test_build_j_deterministic_box_kernel(gpu_ctx, oracle, dims):
    """The TMA box kernel with a dynamic tail and the mbarrier-paired C0
    reduction (256-row tiles / merged classes / KO = 2): repeated sweeps are
    bit-identical."""
    import paper_2403_01778_b200 as r1
    rng = np.random.default_rng(sum(dims))
    a = rng.standard_normal(int(np.prod(dims)))
    f = [rng.standard_normal(k) for k in dims]
    f = [u / np.linalg.norm(u) for u in f]
    t = r1.DenseTensor(dims, a)
    b0 = r1.build_j(t, r1.FactorSet(0.0, f)).blocks
    for _ in range(4):
        assert np.array_equal(r1.build_j(t, r1.FactorSet(0.0, f)).blocks, b0)


def test_dynamic_tail_and_merged_classes_deterministic(gpu_ctx, oracle):
    """A shape that really takes the scheduled dynamic tail (>= 64 panels per
    CTA) and the merged alignment classes (I0 = 136: K = 2, I1 / K = 240), as
    the plan reports it: repeated sweeps bit-identical, and equal to the oracle
    within the contraction bound."""
    import paper_2403_01778_b200 as r1
    dims = (136, 480, 800)
    info = gpu_ctx.sweep_plan_info(dims)
    assert info["K"] > 1 and info["ndyn"] > 0, info
    a = oracle.oracle_random_tensor(dims, 17)
    f = oracle.oracle_random_unit_factors(dims, 18)
    t = r1.DenseTensor(dims, a)
    b0 = r1.build_j(t, r1.FactorSet(0.0, f)).blocks
    for _ in range(3):
        assert np.array_equal(r1.build_j(t, r1.FactorSet(0.0, f)).blocks, b0)
    want = oracle.build_j(a, dims, f)
    scale = oracle.build_j_numpy(np.abs(a), dims, [np.abs(u) for u in f])
    assert np.all(np.abs(b0 - want) <= 1e-13 * scale + 1e-300)


@pytest.mark.parametrize("dims", [(48, 46, 44, 45), (20, 22, 21, 24, 20), (64, 60, 36, 32)])
def test_two_lane_recursion(gpu_ctx, oracle, dims):
    """Tensors large enough (>= 2^22 elements, order >= 4) that the recursion
    forks onto the side stream (root B01 second stage + C1 subtree beside the
    C0 subtree): every block against the oracle, repeats
    bit-identical."""
    import paper_2403_01778_b200 as r1
    assert int(np.prod(dims)) >= 1 << 22
    a = oracle.oracle_random_tensor(dims, 31)
    f = oracle.oracle_random_unit_factors(dims, 32)
    t = r1.DenseTensor(dims, a)
    b0 = r1.build_j(t, r1.FactorSet(0.0, f)).blocks
    for _ in range(2):
        assert np.array_equal(r1.build_j(t, r1.FactorSet(0.0, f)).blocks, b0)
    scale = oracle.build_j_numpy(np.abs(a), dims, [np.abs(u) for u in f])
    assert np.all(np.abs(b0 - oracle.build_j(a, dims, f)) <= 1e-13 * scale + 1e-300)


def test_build_j_errors(gpu_ctx, oracle):
    """nepv.cpp:24-41 / test_nepv.cpp:104-107, 227-232."""
    import paper_2403_01778_b200 as r1
    dims = (3, 3, 3)
    a = r1.DenseTensor(dims, oracle.oracle_random_tensor(dims, 20))
    f = oracle.oracle_random_unit_factors(dims, 21)
    zero = [f[0], f[1], np.zeros(3)]
    with pytest.raises(RuntimeError, match="zero factor for mode 2"):
        r1.build_j(a, r1.FactorSet(0.0, zero))
    with pytest.raises(ValueError, match="not unit length"):
        r1.build_j(a, r1.FactorSet(0.0, [f[0] * 1.5, f[1], f[2]]))
    with pytest.raises(ValueError):
        r1.build_block(a, r1.FactorSet(0.0, f), 1, 1)
    with pytest.raises(ValueError, match="order mismatch"):
        r1.build_j(a, r1.FactorSet(0.0, f[:2]))


MERGE_SHAPES = [(20, 8, 5), (200, 10, 7), (500, 8, 3), (60, 60, 9), (1000, 4, 3), (60, 8, 5, 3),
                (40, 12, 6, 2), (100, 4, 2, 2, 2), (20, 20, 20, 20), (100, 100, 100)]


def test_build_j_merged_classes_forced():
    """Every merged-alignment-class configuration (R1_SWEEP_MERGE=2 forces the
    merged view whenever legal, including tiles holding up to 4 classes) in a
    fresh process on the development build, against the oracle."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = f"""
import numpy as np, sys
sys.path.insert(0, {root!r})
import paper_2403_01778_b200 as r1
from oracle import rank1_oracle as o
ctx = r1.default_context()
for dims in {MERGE_SHAPES!r}:
    a = o.oracle_random_tensor(dims, 5)
    f = o.oracle_random_unit_factors(dims, 6)
    want = o.build_j(a, dims, f)
    got = r1.build_j(r1.DenseTensor(dims, a), r1.FactorSet(0.0, f)).blocks
    scale = o.build_j_numpy(np.abs(a), dims, [np.abs(u) for u in f])
    assert ctx.sweep_plan_info(dims)["K"] > 1 or dims[0] % 16 == 0 or dims[0] % 4, dims
    err = np.max(np.abs(got - want) / (scale + 1e-300))
    assert err <= 1e-13, (dims, err)
print("ok")
"""
    dev_lib = os.path.join(root, "paper_2403_01778_b200", "librank1_b200_dev.so")
    if not os.path.exists(dev_lib):
        pytest.skip("development build not present (build.py --dev)")
    # the switch exists only in the development build
    env = dict(os.environ, R1_SWEEP_MERGE="2", R1_LIB_PATH=dev_lib)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr
