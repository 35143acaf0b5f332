"""Multi-GPU HOSCF / iHOSCF: contiguous slabs along the slowest
(last) mode, one process per GPU — a thin Python layer over the C-ABI.

The work is all in the library (csrc/comm.cu, csrc/solver.cu):
  * r1_build_j_sharded: the rank's slab sweep (its slice of the last factor is
    read in place) + ONE NCCL group per sweep — all-reduce of the partial
    blocks (m, n < d-1), all-gather / per-root broadcast of the blocks (m, d-1)
    straight into their column runs of the global block;
  * r1_solve_sharded: the C++ HOSCF / iHOSCF driver (solvers.cpp:129-297 control
    flow) with that sweep; eigen step, RQI and the device stopping test run
    replicated on the identical bits NCCL returns to every rank.
This module only joins the ranks (the NCCL unique id travels over the caller's
torch.distributed group) and mirrors the slab / exchange plan for the tests.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np


def slab_bounds(extent: int, world: int, rank: int) -> tuple[int, int]:
    """[lo, hi) of rank's slab: sizes differ by at most one, larger first
    (r1_slab_bounds)."""
    base, rem = divmod(extent, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def pairs(d: int):
    return [(m, n) for m in range(d) for n in range(m + 1, d)]


def local_dims(dims, lo: int, hi: int):
    return tuple(list(dims[:-1]) + [hi - lo])


@dataclass
class ExchangeOp:
    m: int
    n: int
    local_off: int     # element offset in the rank's local (slab) block buffer
    global_off: int    # element offset in the global block buffer
    local_count: int   # elements of the local block
    gathered: bool     # n == d-1: columns gathered, else partial sums all-reduced


def exchange_plan(dims, world: int, rank: int) -> list[ExchangeOp]:
    """The library's plan for this rank (r1x_exchange_plan, csrc/comm.cu)."""
    from . import _lib
    d = len(dims)
    out = np.zeros(6 * d * d, dtype=np.int64)
    gd = _lib.dims_arr(dims)
    _lib.check(_lib.lib().r1x_exchange_plan(_lib.u64p(gd), d, world, rank,
                                            out.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                            d * d))
    return [ExchangeOp(int(o[0]), int(o[1]), int(o[2]), int(o[3]), int(o[4]), bool(o[5]))
            for o in out.reshape(-1, 6)[:len(pairs(d))]]


def exchange_numpy(local_list, dims):
    """The collectives of the plan applied to every rank's local blocks at once
    (all-reduce = sum, gather = place each rank's run): the global blocks."""
    world = len(local_list)
    total = sum(dims[m] * dims[n] for m, n in pairs(len(dims)))
    out = np.zeros(total)
    for r in range(world):
        lo, hi = slab_bounds(dims[-1], world, r)
        for op in exchange_plan(dims, world, r):
            src = local_list[r][op.local_off:op.local_off + op.local_count]
            if op.gathered:
                rows = dims[op.m]
                out[op.global_off + rows * lo:op.global_off + rows * hi] = src
            else:
                out[op.global_off:op.global_off + op.local_count] += src
    return out


def exchange_torch(local, dims, world: int, rank: int, dist, out):
    """The same plan executed with torch.distributed collectives (the CPU
    multi-process tests drive it over gloo; the library issues the identical
    operations through NCCL): all-reduce into the partial blocks, one broadcast
    per root into its column run of each gathered block."""
    for op in exchange_plan(dims, world, rank):
        if not op.gathered:
            seg = out[op.global_off:op.global_off + op.local_count]
            seg.copy_(local[op.local_off:op.local_off + op.local_count])
            dist.all_reduce(seg)
            continue
        rows = dims[op.m]
        for r in range(world):
            rlo, rhi = slab_bounds(dims[-1], world, r)
            if rhi == rlo:
                continue
            dst = out[op.global_off + rows * rlo:op.global_off + rows * rhi]
            if r == rank:
                dst.copy_(local[op.local_off:op.local_off + op.local_count])
            dist.broadcast(dst, src=r)
    return out


class Comm:
    """An NCCL communicator attached to a context (r1_comm_init)."""

    def __init__(self, handle, world: int, rank: int):
        self.handle = handle
        self.world = world
        self.rank = rank

    def close(self):
        from . import _lib
        if self.handle:
            _lib.lib().r1_comm_destroy(self.handle)
            self.handle = None


def init_comm(ctx, dist, world: int, rank: int) -> Comm:
    """Join the ranks of `dist` (an initialised torch.distributed group, any
    backend) in one NCCL communicator attached to `ctx`: rank 0 makes the id,
    the group broadcasts it."""
    import torch

    from . import _lib
    L = _lib.lib()
    idb = (ctypes.c_char * 128)()
    if rank == 0:
        _lib.check(L.r1_comm_unique_id(idb))
    if world > 1:
        t = torch.frombuffer(bytearray(idb.raw), dtype=torch.uint8).clone()
        if dist.get_backend() == "nccl":
            t = t.cuda()
        dist.broadcast(t, src=0)
        idb = (ctypes.c_char * 128).from_buffer_copy(bytes(t.cpu().numpy().tobytes()))
    h = ctypes.c_void_p()
    _lib.check(L.r1_comm_init(ctx.handle, world, rank, idb, ctypes.byref(h)))
    return Comm(h, world, rank)


def build_j_sharded(ctx, slab, dims, factors_dev_ptr: int, blocks_dev_ptr: int, fro2_dev_ptr=None):
    """One sharded sweep: global blocks (identical on every rank) from this
    rank's slab (r1_build_j_sharded)."""
    from . import _lib
    gd = _lib.dims_arr(dims)
    _lib.check(_lib.lib().r1_build_j_sharded(ctx.handle, slab.handle, _lib.u64p(gd), len(dims),
                                             ctypes.c_void_p(factors_dev_ptr),
                                             ctypes.c_void_p(blocks_dev_ptr),
                                             ctypes.c_void_p(fro2_dev_ptr) if fro2_dev_ptr else None))


def solve_distributed(algorithm, slab, dims, opts, ctx=None):
    """hoscf | ihoscf on a tensor sharded in slabs along its last mode
    (r1_solve_sharded).  slab: this rank's DeviceTensor; dims: global dims.  The
    context must carry a communicator (init_comm).  Returns the reference-
    shaped SolveReport, identical on every rank."""
    from . import InvalidArgument, solve
    if algorithm not in ("hoscf", "ihoscf"):
        raise InvalidArgument("sharded solves support hoscf and ihoscf: " + algorithm)
    return solve(algorithm, slab, opts, ctx, global_dims=dims)
