"""CPU-suite checks of the drop-in boundary and the host-side logic:
  * librank1_b200.so loads and exports every symbol include/rank1_b200.h declares;
  * without a GPU every device entry point fails loudly (no CPU fallback);
  * option defaults equal the reference's SolveOptions (solvers.hpp:17-31);
  * the Python mirror's host-side pieces (split/stack, SymBlockMatrix,
    DenseTensor validation) reproduce the reference KATs (test_nepv.cpp:16-57)."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "rank1_b200.h")


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(r1_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2403_01778_b200 import _lib
    lib = ctypes.CDLL(_lib.LIB_PATH)
    names = header_functions()
    assert len(names) >= 25
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert set(names) <= set(_lib.SIGNATURES) | {"r1_generate_config"}


def test_abi_version_and_sizes():
    from paper_2403_01778_b200 import _lib
    L = _lib.lib()
    assert L.r1_abi_version() == 1
    d = _lib.dims_arr([3, 4, 5])
    assert L.r1_blocks_numel(_lib.u64p(d), 3) == 3 * 4 + 3 * 5 + 4 * 5


def test_option_defaults_match_reference():
    import paper_2403_01778_b200 as r1
    from paper_2403_01778_b200 import _lib
    c = _lib.SolveOptionsC()
    _lib.lib().r1_solve_options_default(ctypes.byref(c))
    py = r1.SolveOptions()
    assert c.tol == py.tol == 1e-4
    assert c.max_iters == py.max_iters == 500
    assert c.seed == py.seed == 0 and c.init == 0 and py.init == "uniform01"
    assert c.determinism == 1 and py.determinism
    assert c.record_kkt == 1 and py.record_kkt
    assert c.rqi_accept_rule == 0 and py.rqi_accept_rule == "magnitude"
    assert c.reuse_intermediates == 0 and c.scf_lambda_rtol == 0.0


def _no_gpu():
    try:
        import torch
        return not torch.cuda.is_available()
    except Exception:
        return True


@pytest.mark.skipif(not _no_gpu(), reason="GPU present")
def test_device_entry_points_fail_loudly_without_gpu():
    import paper_2403_01778_b200 as r1
    from paper_2403_01778_b200 import _lib
    h = ctypes.c_void_p()
    rc = _lib.lib().r1_context_create(0, ctypes.byref(h))
    assert rc == _lib.R1_ERR_NO_DEVICE
    assert b"no CPU fallback" in _lib.lib().r1_last_error()
    with pytest.raises(r1.DeviceError):
        r1.build_j(r1.DenseTensor([2, 2, 2], np.ones(8)), r1.FactorSet(0.0, [[1.0, 0.0]] * 3),
                   ctx=None)


def test_split_and_stack_kats():
    """test_nepv.cpp:16-57 on the host mirror."""
    import paper_2403_01778_b200 as r1
    from oracle import rank1_oracle as O
    f = O.oracle_random_unit_factors((3, 4, 2), 1)
    x = r1.stack_factors(r1.FactorSet(0.0, f))
    assert abs(x.norm() - 1.0) <= 1e-14
    r = r1.split_factors(x)
    assert not r.any_degenerate()
    for u, v in zip(r.factors.factors, f):
        np.testing.assert_allclose(u, v, rtol=1e-12)
    z = r1.StackedVector([2, 3], [0.6, 0.8, 0.0, 0.0, 0.0])
    rz = r1.split_factors(z)
    assert rz.degenerate == [0, 1] and not rz.factors.factors[1].any()
    f4 = O.oracle_random_unit_factors((2, 3, 2, 4), 2)
    x4 = r1.stack_factors(r1.FactorSet(0.0, f4))
    for n in range(4):
        assert abs(x4.block_norm(n) - 0.5) <= 1e-14
    bad = [f4[0], f4[1] * 1.5, f4[2], f4[3]]
    with pytest.raises(ValueError):
        r1.stack_factors(r1.FactorSet(0.0, bad))


def test_symblockmatrix_host_ops_match_oracle():
    import paper_2403_01778_b200 as r1
    from oracle import rank1_oracle as O
    dims = (3, 2, 4, 2)
    a = O.oracle_random_tensor(dims, 11)
    f = O.oracle_random_unit_factors(dims, 12)
    blocks = O.build_j(a, dims, f)
    j = r1.SymBlockMatrix(dims, blocks)
    d = j.dense()
    assert np.array_equal(d, d.T)
    x = O.oracle_random_unit(j.total_dim(), 13)
    np.testing.assert_allclose(j.matvec(x), d @ x, rtol=1e-12, atol=1e-14)
    assert abs(j.frobenius_norm() - np.linalg.norm(d)) <= 1e-12 * np.linalg.norm(d)
    assert j.scale() == 1.0 / 3
    with pytest.raises(ValueError):
        j.block(2, 1)


def test_dense_tensor_validation():
    import paper_2403_01778_b200 as r1
    with pytest.raises(ValueError):
        r1.DenseTensor([2, 0, 3])
    with pytest.raises(ValueError):
        r1.DenseTensor([2, 3], np.zeros(5))
    t = r1.DenseTensor([2, 3])
    assert t.order() == 2 and t.size() == 6 and t.dim(1) == 3
    assert r1.solver_names() == ["hoscf", "ihoscf", "hopm", "jacobi_hopm", "asvd", "jacobi_asvd"]
