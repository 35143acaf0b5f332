#!/usr/bin/env python3
"""Randomised parity of the TWO-LANE sweep (orders 4-6, 4-16 M elements: the
sizes that fork the recursion onto the side stream) against the oracle's
restatement, each shape swept three times (bit-identical repeats).
    python tools/fork_fuzz_probe.py [seconds] [seed]"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_01778_b200 as r1  # noqa: E402
from oracle import rank1_oracle as O  # noqa: E402

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 3)
O.build()
t0 = time.time()
n_ok, bad = 0, []
while time.time() - t0 < budget:
    d = int(rng.integers(4, 7))
    target = float(rng.uniform(4.2e6, 1.6e7))
    while True:
        dims = [int(rng.integers(2, {4: 120, 5: 40, 6: 20}[d])) for _ in range(d)]
        scale = (target / np.prod(dims)) ** (1.0 / d)
        dims = tuple(max(2, int(round(k * scale))) for k in dims)
        if 4.2e6 <= np.prod(dims) <= 2.0e7:
            break
    if rng.random() < 0.4:
        dims = tuple(max(2, (k // 4) * 4) for k in dims)
        if np.prod(dims) < (1 << 22):
            continue
    a = O.oracle_random_tensor(dims, int(rng.integers(1 << 30)))
    f = O.oracle_random_unit_factors(dims, int(rng.integers(1 << 30)))
    try:
        t = r1.DenseTensor(dims, a)
        got = r1.build_j(t, r1.FactorSet(0.0, f)).blocks
        for _ in range(2):
            if not np.array_equal(r1.build_j(t, r1.FactorSet(0.0, f)).blocks, got):
                bad.append(("repeat", dims))
    except Exception:
        print("build_j FAILED at dims", dims, flush=True)
        raise
    want = O.build_j(a, dims, f)
    scale_b = O.build_j_numpy(np.abs(a), dims, [np.abs(u) for u in f])
    if not np.all(np.abs(got - want) <= 1e-13 * scale_b + 1e-300):
        bad.append(("parity", dims))
    n_ok += 1
print(f"fork fuzz: {n_ok} shapes, {len(bad)} failures in {time.time() - t0:.0f} s", bad[:10])
