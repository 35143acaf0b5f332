"""CPU: the compiled reference's own iteration-count sensitivity on the
stagnating iHOSCF cases of tests/test_solver_gpu.py (CHAOTIC).  One-ulp
perturbations of the input (each entry times 1 + {-1, 0, 1} 2^-52) move the
reference's iteration count by several iterations — the rounding-level noise
floor any reimplementation is measured against."""
import numpy as np
import pytest


@pytest.mark.parametrize("dims,kind,lo_span", [((20, 20, 20), "c1", 3), ((7, 5, 9), "gauss", 3)])
def test_reference_iteration_count_is_rounding_sensitive(oracle, ref, dims, kind, lo_span):
    a = oracle.gen_config(1, dims, 1) if kind == "c1" else oracle.oracle_random_tensor(dims, 11)
    rng = np.random.default_rng(0)
    its = []
    for t in range(12):
        b = a.copy() if t == 0 else a * (1 + rng.choice([-1, 0, 1], size=a.size) * 2.0 ** -52)
        its.append(ref.solve("ihoscf", b, dims, tol=1e-10, max_iters=500, seed=1)["iterations"])
    assert max(its) - min(its) >= lo_span, its
    # HOSCF on the same inputs is not sensitive
    hits = {ref.solve("hoscf", a * (1 + rng.choice([-1, 0, 1], size=a.size) * 2.0 ** -52), dims,
                      tol=1e-10, max_iters=500, seed=1)["iterations"] for _ in range(4)}
    assert len(hits) <= 2
