"""The alternative paths behind the development switches stay
correct: each runs in a fresh process (the switches are read once) on the
DEVELOPMENT build (librank1_b200_dev.so: the release library ignores the
environment) against the compiled reference / numpy."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHECK = f"""
import numpy as np, sys
sys.path.insert(0, {ROOT!r})
import paper_2403_01778_b200 as r1
from oracle import ref
ctx = r1.default_context()
# RQI (BK factor + solve) against the reference
for n in (40, 333, 700):
    rng = np.random.default_rng(n)
    m = rng.standard_normal((n, n))
    s = m + m.T
    x = rng.standard_normal(n)
    x /= np.linalg.norm(x)
    y, yr = r1.rayleigh_quotient_step(s, x), ref.rayleigh_quotient_step(s, x)
    assert (y is None) == (yr is None), n
    if y is not None:
        assert min(np.max(np.abs(y - yr)), np.max(np.abs(y + yr))) <= 1e-8, n
# eigen step on block operators (small n: cluster or grid kernel) against numpy
for dims in ((3, 4, 2), (20, 30, 25), (60, 60, 60), (500, 600, 50)):
    rng = np.random.default_rng(sum(dims))
    a = rng.standard_normal(int(np.prod(dims)))
    f = [rng.standard_normal(k) for k in dims]
    f = [u / np.linalg.norm(u) for u in f]
    j = r1.build_j(r1.DenseTensor(dims, a), r1.FactorSet(0.0, f))
    w = np.linalg.eigvalsh(j.dense())
    want = w[0] if abs(w[0]) > abs(w[-1]) * (1 + 1e-12) else w[-1]
    p, _ = r1.eig_blocks(j)
    assert abs(p.value - want) <= 1e-11 * abs(want), (dims, p.value, want)
# a full iHOSCF solve against the reference
dims = (30, 30, 30)
a = ref.generate("exp", dims)
got = r1.ihoscf(r1.DenseTensor(dims, a), r1.SolveOptions(tol=1e-8))
want = ref.solve("ihoscf", a, dims, tol=1e-8, max_iters=500, seed=0)
assert got.converged and abs(got.result.lambda_ - want["lam"]) <= 1e-10 * want["lam"]
# sweep (every block) against the oracle restatement
from oracle import rank1_oracle as o
for dims in ((200, 200, 7), (200, 64, 6, 5), (1000, 4, 3), (60, 60, 12, 5, 4), (136, 480, 40), (72, 500, 11)):
    a = o.oracle_random_tensor(dims, 3)
    f = o.oracle_random_unit_factors(dims, 4)
    got = r1.build_j(r1.DenseTensor(dims, a), r1.FactorSet(0.0, f)).blocks
    scale = o.build_j_numpy(np.abs(a), dims, [np.abs(u) for u in f])
    assert np.all(np.abs(got - o.build_j(a, dims, f)) <= 1e-13 * scale + 1e-300), dims
print("ok")
"""


DEV_LIB = os.path.join(ROOT, "paper_2403_01778_b200", "librank1_b200_dev.so")


@pytest.mark.parametrize("env", [{"R1_SOLVER_GRAPHS": "0"}, {"R1_BK_GRID_SOLVE": "1"},
                                 {"R1_EIG_SMALL": "0"}, {"R1_EIG_CLUSTER": "8"}, {"R1_EIG_TILED": "0"},
                                 {"R1_SWEEP_NRA8": "0"}, {"R1_SWEEP_MERGE": "0"},
                                 {"R1_SWEEP_WIDE": "0"}, {"R1_SWEEP_FORK": "0"}, {"R1_SWEEP_FORK": "1"},
                                 {"R1_SWEEP_NS": "4", "R1_SWEEP_NS_MINP": "0"}])
def test_switch_paths(gpu_ctx, env):
    if not os.path.exists(DEV_LIB):
        pytest.skip("development build not present (build.py --dev)")
    env = dict(env, R1_LIB_PATH=DEV_LIB)
    r = subprocess.run([sys.executable, "-c", CHECK], env=dict(os.environ, **env), capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout[-2000:] + r.stderr[-3000:]
