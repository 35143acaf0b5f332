"""The N > 1 path on CPU: world_size-2 (and 3, uneven slabs) gloo process
groups run the real slab exchange (paper_2403_01778_b200.distributed.exchange:
all-reduce of partial blocks, all-gather of blocks touching the sharded mode)
on per-rank local blocks computed by the oracle for each rank's slab; the
assembled blocks must equal the oracle's blocks of the whole tensor."""
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
        from paper_2403_01778_b200.distributed import exchange, local_dims, slab_bounds
        a = O.oracle_random_tensor(dims, seed).reshape(dims, order="F")
        f = O.oracle_random_unit_factors(dims, seed + 1)
        lo, hi = slab_bounds(dims[-1], world, rank)
        ld = local_dims(dims, lo, hi)
        slab = np.ascontiguousarray(a[..., lo:hi].reshape(-1, order="F"))
        fl = list(f[:-1]) + [f[-1][lo:hi]]
        local = torch.from_numpy(O.build_j_numpy(slab, ld, fl))
        nb = sum(dims[m] * dims[n] for m in range(len(dims)) for n in range(m + 1, len(dims)))
        out = torch.zeros(nb, dtype=torch.float64)
        exchange(local, dims, world, rank, dist, out)
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


def test_driver_init_factors_match_reference():
    """The distributed driver's uniform01 init (solvers.cpp:34-49) equals the
    oracle's (pinned to the reference)."""
    from oracle import rank1_oracle as O
    from paper_2403_01778_b200.distributed import random_unit_factors
    for dims, seed in [((4, 5, 6), 3), ((10, 2), 0)]:
        for a, b in zip(random_unit_factors(dims, seed, 2), O.random_unit_factors(dims, seed, 2)):
            np.testing.assert_allclose(a, b, rtol=1e-15)
