#!/usr/bin/env python3
"""Randomised parity sweep (development tool): build_j against the oracle's
restatement (bit-pinned to the reference) on random shapes of orders 2-6, and
HOSCF / iHOSCF against the compiled reference on random small tensors.
    python tools/fuzz_probe.py [seconds] [seed]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_01778_b200 as r1  # noqa: E402
from oracle import rank1_oracle as O  # noqa: E402
from oracle import ref  # noqa: E402

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 7)
mode = sys.argv[3] if len(sys.argv) > 3 else ""  # "solves" / "hoscf": skip the sweep checks, solve every case; "sweeps": no solves
solves_only = mode in ("solves", "hoscf")
O.build()
t0 = time.time()
nb = ns = 0
bad = []
diffs = []
while time.time() - t0 < budget:
    d = int(rng.integers(2, 7))
    cap = {2: 700, 3: 160, 4: 40, 5: 16, 6: 9}[d]
    dims = tuple(int(rng.integers(1, cap + 1)) for _ in range(d))
    if rng.random() < 0.3:  # aligned sizes (merged classes, 16-row tiles)
        dims = tuple(max(1, (k // 8) * 8) for k in dims)
    a = O.oracle_random_tensor(dims, int(rng.integers(1 << 30)))
    f = O.oracle_random_unit_factors(dims, int(rng.integers(1 << 30)))
    if not solves_only:
        try:
            got = r1.build_j(r1.DenseTensor(dims, a), r1.FactorSet(0.0, f)).blocks
        except Exception:
            print("build_j FAILED at dims", dims, "after", nb, "sweeps", flush=True)
            raise
        want = O.build_j(a, dims, f)
        scale = O.build_j_numpy(np.abs(a), dims, [np.abs(u) for u in f])
        if not np.all(np.abs(got - want) <= 1e-13 * scale + 1e-300):
            bad.append(("build_j", dims))
        nb += 1
    do_solve = solves_only or rng.random() < 0.25  # (drawn in every mode: same shape sequence)
    if mode == "sweeps":
        continue
    if d >= 3 and np.prod(dims) <= 2e5 and min(dims) >= 2 and do_solve:
        alg = "hoscf" if mode == "hoscf" else ("ihoscf" if solves_only or rng.random() < 0.5 else "hoscf")
        seed = int(rng.integers(100))
        rep = r1.solve(alg, r1.DenseTensor(dims, a), r1.SolveOptions(tol=1e-10, max_iters=300, seed=seed))
        w = ref.solve(alg, a, dims, tol=1e-10, max_iters=300, seed=seed)
        ok = abs(rep.result.lambda_ - w["lam"]) <= 1e-9 * max(1.0, abs(w["lam"]))
        ok = ok and (abs(rep.iterations - w["iterations"]) <= 1 or not w["converged"])
        if not ok:
            bad.append((alg, dims, seed, rep.iterations, w["iterations"], rep.result.lambda_, w["lam"]))
        diffs.append(rep.iterations - w["iterations"])
        ns += 1
print(f"fuzz: {nb} sweeps, {ns} solves, {len(bad)} mismatches in {time.time() - t0:.0f} s")
if diffs:
    dd = np.array(diffs)
    print(f"iteration count device - reference: mean {dd.mean():+.2f}, |d| <= 1 in {np.mean(np.abs(dd) <= 1):.0%}, "
          f"> +1 in {np.mean(dd > 1):.0%}, < -1 in {np.mean(dd < -1):.0%}")
for b in bad[:20]:
    print("  ", b)
