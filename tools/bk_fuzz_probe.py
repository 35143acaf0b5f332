#!/usr/bin/env python3
"""Randomised check of the hand-written Bunch-Kaufman (csrc/bk.cu) against the
compiled reference's ldlt (sym_eig.cpp:233-407): sizes around and across the
32-column panels, random / zero-diagonal / tiny-diagonal / diagonally
dominant / shifted-block matrices; the pivot sequence bit-equal, D within
1e-10, the condition estimate within 1e-8 (development tool).
    python tools/bk_fuzz_probe.py [seconds] [seed]"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2403_01778_b200 as r1  # noqa: E402
from oracle import ref  # noqa: E402
from test_bk_gpu import dev_ldlt, ref_d  # noqa: E402

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 5)
ctx = r1.default_context()
t0 = time.time()
cnt, bad = 0, []
while time.time() - t0 < budget:
    n = int(rng.choice([int(rng.integers(1, 130)), 32 * int(rng.integers(1, 30)) + int(rng.integers(-2, 3)),
                        int(rng.integers(130, 1300))]))
    n = max(1, n)
    kind = ["rand", "zero_diag", "tiny_diag", "dominant", "lowrank_shift"][int(rng.integers(5))]
    m = rng.standard_normal((n, n))
    s = m + m.T
    if kind == "zero_diag":
        np.fill_diagonal(s, 0.0)
    elif kind == "tiny_diag":
        np.fill_diagonal(s, 1e-3 * rng.standard_normal(n))
    elif kind == "dominant":
        s += np.diag(rng.choice([-1, 1], n) * 3.0 * np.sqrt(n))
    elif kind == "lowrank_shift":
        u = rng.standard_normal((n, min(n, 6)))
        s = u @ np.diag(rng.standard_normal(min(n, 6)) * 5) @ u.T + 1e-3 * s - 0.7 * np.eye(n)
    ipiv, diag, sub, sing, cond = dev_ldlt(ctx, s)
    w, ipr, singr, condr = ref.ldlt(s)
    ok = sing == singr and np.array_equal(ipiv, ipr)
    if ok and not sing:
        dr, sr = ref_d(w, ipr)
        sc = np.max(np.abs(s))
        ok = np.max(np.abs(diag - dr)) <= 1e-10 * sc and np.max(np.abs(sub - sr)) <= 1e-10 * sc
        if np.isfinite(condr):
            ok = ok and abs(cond - condr) <= 1e-8 * condr
    if not ok:
        first = np.nonzero(ipiv != ipr)[0][:3] if len(ipiv) == len(ipr) else None
        bad.append((n, kind, sing, singr, first))
    cnt += 1
print(f"bk fuzz: {cnt} factorisations, {len(bad)} mismatches in {time.time() - t0:.0f} s")
for b in bad[:10]:
    print("  ", b)
