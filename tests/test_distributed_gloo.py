"""The N > 1 path on CPU: world_size-2 (and 3, uneven slabs) gloo process
groups execute the library's exchange plan (r1x_exchange_plan, csrc/comm.cu —
the same all-reduces and per-root column-run broadcasts the library issues
through NCCL) on per-rank local blocks computed by the oracle for each rank's
slab; the assembled blocks must equal the oracle's blocks of the whole tensor,
bit-identical on every rank."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, dims, seed, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import rank1_oracle as O
        from paper_2403_01778_b200.distributed import exchange_torch, local_dims, slab_bounds
        a = O.oracle_random_tensor(dims, seed).reshape(dims, order="F")
        f = O.oracle_random_unit_factors(dims, seed + 1)
        lo, hi = slab_bounds(dims[-1], world, rank)
        ld = local_dims(dims, lo, hi)
        slab = np.ascontiguousarray(a[..., lo:hi].reshape(-1, order="F"))
        fl = list(f[:-1]) + [f[-1][lo:hi]]
        local = torch.from_numpy(O.build_j_numpy(slab, ld, fl))
        nb = sum(dims[m] * dims[n] for m in range(len(dims)) for n in range(m + 1, len(dims)))
        out = torch.zeros(nb, dtype=torch.float64)
        exchange_torch(local, dims, world, rank, dist, out)
        q.put((rank, out.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,dims", [(2, (7, 5, 10)), (3, (6, 5, 4, 7)), (2, (4, 9)),
                                        (3, (5, 4, 3, 2, 8))])
def test_slab_exchange_matches_full_sweep(world, dims):
    from oracle import rank1_oracle as O
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, dims, 5, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    a = O.oracle_random_tensor(dims, 5)
    f = O.oracle_random_unit_factors(dims, 6)
    want = O.build_j_numpy(a, dims, f)
    for r in range(world):
        np.testing.assert_allclose(res[r], want, rtol=1e-12, atol=1e-12)
    # every rank holds identical bits (replicated eigen step inputs)
    for r in range(1, world):
        assert np.array_equal(res[r], res[0])


def test_slab_bounds_partition():
    from paper_2403_01778_b200.distributed import slab_bounds
    for extent in (1, 7, 60, 125, 1000, 4000):
        for world in (1, 2, 3, 4, 8):
            spans = [slab_bounds(extent, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == extent
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))
            sizes = [h - l for l, h in spans]
            assert max(sizes) - min(sizes) <= 1


def test_exchange_numpy_reference():
    from oracle import rank1_oracle as O
    from paper_2403_01778_b200.distributed import exchange_numpy, local_dims, slab_bounds
    dims = (5, 6, 9)
    a = O.oracle_random_tensor(dims, 3).reshape(dims, order="F")
    f = O.oracle_random_unit_factors(dims, 4)
    locs = []
    for r in range(4):
        lo, hi = slab_bounds(dims[-1], 4, r)
        slab = np.ascontiguousarray(a[..., lo:hi].reshape(-1, order="F"))
        locs.append(O.build_j_numpy(slab, local_dims(dims, lo, hi), list(f[:-1]) + [f[-1][lo:hi]]))
    np.testing.assert_allclose(exchange_numpy(locs, dims),
                               O.build_j_numpy(a.reshape(-1, order="F"), dims, f), rtol=1e-12, atol=1e-12)


def test_slab_bounds_match_library():
    import ctypes

    from paper_2403_01778_b200 import _lib
    from paper_2403_01778_b200.distributed import slab_bounds
    lo, hi = ctypes.c_uint64(), ctypes.c_uint64()
    for extent in (3, 60, 125, 4000):
        for world in (1, 2, 3, 8):
            for r in range(world):
                _lib.check(_lib.lib().r1_slab_bounds(extent, world, r, ctypes.byref(lo), ctypes.byref(hi)))
                assert (lo.value, hi.value) == slab_bounds(extent, world, r)


def test_exchange_plan_layout():
    """Local offsets follow the slab's own pair order, global offsets the whole
    tensor's; gathered blocks are exactly the pairs (m, d-1)."""
    from paper_2403_01778_b200.distributed import exchange_plan, local_dims, pairs, slab_bounds
    dims = (4, 3, 5, 11)
    for world in (1, 2, 4):
        for r in range(world):
            lo, hi = slab_bounds(dims[-1], world, r)
            ld = local_dims(dims, lo, hi)
            ops = exchange_plan(dims, world, r)
            loff = goff = 0
            for op, (m, n) in zip(ops, pairs(4)):
                assert (op.m, op.n) == (m, n) and op.gathered == (n == 3)
                assert op.local_off == loff and op.global_off == goff
                assert op.local_count == ld[m] * ld[n]
                loff += ld[m] * ld[n]
                goff += dims[m] * dims[n]
