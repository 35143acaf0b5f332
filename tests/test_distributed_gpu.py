"""The distributed HOSCF / iHOSCF driver (paper_2403_01778_b200.distributed.
solve_distributed: slab sweep + exchange + replicated eigen / RQI / stopping
test) on one GPU (world = 1) against the single-GPU solver and the reference;
the N > 1 exchange itself is covered by tests/test_distributed_gloo.py."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("alg,dims,kind,tol,seed", [
    ("hoscf", (30, 30, 30), "exp", 1e-4, 0), ("ihoscf", (30, 30, 30), "exp", 1e-4, 0),
    ("hoscf", (7, 5, 9), "gauss", 1e-10, 1), ("ihoscf", (7, 5, 9), "gauss", 1e-10, 1),
    ("hoscf", (6, 5, 4, 3), "gauss", 1e-8, 3), ("ihoscf", (10, 10, 10, 10, 10), "tan", 1e-4, 0)])
def test_distributed_driver_matches_single_gpu(gpu_ctx, oracle, ref, alg, dims, kind, tol, seed):
    import paper_2403_01778_b200 as r1
    from paper_2403_01778_b200.distributed import solve_distributed
    a = ref.generate(kind, dims) if kind in ("exp", "tan") else oracle.oracle_random_tensor(dims, 11)
    o = r1.SolveOptions(tol=tol, max_iters=500, seed=seed)
    t = r1.DeviceTensor.from_host(a, dims)
    got = solve_distributed(alg, t, dims, o)
    one = r1.solve(alg, t, o)
    want = ref.solve(alg, a, dims, tol=tol, max_iters=500, seed=seed)
    assert got.converged == want["converged"] == one.converged
    # iHOSCF near stagnation: the RQI accept test |rho_y| > |rho_mid| is a
    # near-tie that flips with last-bit differences (host-side post step here),
    # as for the CHAOTIC cases of test_solver_gpu.py
    slack = 3 if alg == "ihoscf" else 1
    if (alg, dims, kind) == ("ihoscf", (7, 5, 9), "gauss"):
        slack = 6  # the CHAOTIC case of test_solver_gpu.py: stagnates at ~1e-10
    assert abs(got.iterations - want["iterations"]) <= slack
    assert abs(got.iterations - one.iterations) <= slack
    assert abs(got.result.lambda_ - want["lam"]) <= 1e-10 * abs(want["lam"])
    assert abs(got.lambda0 - want["lambda0"]) <= 1e-12 * max(1.0, abs(want["lambda0"]))
    if got.iterations == want["iterations"]:
        for u, v in zip(got.result.factors, want["factors"]):
            assert min(np.max(np.abs(u - v)), np.max(np.abs(u + v))) <= 1e-8
