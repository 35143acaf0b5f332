"""GPU stress: the message-passing kernels (BK panel / cluster solve, small-n
Lanczos) must give bit-identical results run after run (development tool)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_01778_b200 as r1  # noqa: E402
from oracle import rank1_oracle as o  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
# C2-like structured J - rho I at n = 3000 (zero diagonal blocks, planted rank one)
dims = (1000, 1000, 1000)
rng = np.random.default_rng(5)
f = [rng.standard_normal(k) for k in dims]
f = [u / np.linalg.norm(u) for u in f]
blocks = []
for m, n in ((0, 1), (0, 2), (1, 2)):
    k = 3 - m - n
    b = 10.0 * np.outer(f[m], f[n]) * f[k].sum() * 0.03 + 1e-3 * rng.standard_normal((dims[m], dims[n]))
    blocks.append(b)
N = sum(dims)
s = np.zeros((N, N))
offs = [0, 1000, 2000]
for (m, n), b in zip(((0, 1), (0, 2), (1, 2)), blocks):
    s[offs[m]:offs[m] + dims[m], offs[n]:offs[n] + dims[n]] = b * 0.5
    s[offs[n]:offs[n] + dims[n], offs[m]:offs[m] + dims[m]] = b.T * 0.5
x = np.concatenate(f) / np.sqrt(3)
first = r1.rayleigh_quotient_step(s, x)
bad = 0
for i in range(reps):
    y = r1.rayleigh_quotient_step(s, x)
    if (y is None) != (first is None) or (y is not None and not np.array_equal(y, first)):
        bad += 1
print("rqi n=3000 structured: reps", reps, "mismatches", bad, flush=True)
# small-n Lanczos (cluster kernel) through full C1-style solves
d1 = (100, 100, 100)
a = o.oracle_random_tensor(d1, 9)
ref = r1.hoscf(r1.DenseTensor(d1, a), r1.SolveOptions(tol=1e-12, seed=1))
bad = 0
for i in range(reps):
    g = r1.hoscf(r1.DenseTensor(d1, a), r1.SolveOptions(tol=1e-12, seed=1))
    if g.iterations != ref.iterations or g.result.lambda_ != ref.result.lambda_:
        bad += 1
print("hoscf 100^3: reps", reps, "mismatches", bad, flush=True)
