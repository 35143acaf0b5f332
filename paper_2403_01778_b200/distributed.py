"""Multi-GPU sweep: contiguous slabs along the slowest mode.

Rank r holds A[..., lo_r:hi_r] (reference mode d-1, the slowest, is split).
Its local sweep over that slab yields, for every pair (m, n):
  * n <  d-1: a PARTIAL block (sum over the rank's slab)  -> all-reduce(sum)
  * n == d-1: the block's COMPLETE columns lo_r:hi_r       -> all-gather
Block (m, d-1) is column-major I_m x I_{d-1}, so a rank's columns are one
contiguous run: the gather is a plain concatenation (uneven slabs are padded
to the largest slab and compacted).  NCCL gives every rank the same reduced
bits, so the replicated eigen step sees identical inputs on all ranks.

Only host logic lives here (slab bounds, the exchange plan, the exchange
itself over torch.distributed); the per-rank sweep is the device kernel.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def slab_bounds(extent: int, world: int, rank: int) -> tuple[int, int]:
    """[lo, hi) of rank's slab: sizes differ by at most one, larger first."""
    base, rem = divmod(extent, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def pairs(d: int):
    return [(m, n) for m in range(d) for n in range(m + 1, d)]


@dataclass
class BlockSlot:
    m: int
    n: int
    offset: int        # element offset in the global block buffer
    rows: int
    cols: int
    gathered: bool     # n == d-1: columns are gathered, else partial sums reduced


def exchange_plan(dims) -> list[BlockSlot]:
    d = len(dims)
    out, off = [], 0
    for m, n in pairs(d):
        out.append(BlockSlot(m, n, off, dims[m], dims[n], n == d - 1))
        off += dims[m] * dims[n]
    return out


def local_dims(dims, lo: int, hi: int):
    return tuple(list(dims[:-1]) + [hi - lo])


def local_offsets(ldims) -> dict:
    offs, o = {}, 0
    for m, n in pairs(len(ldims)):
        offs[(m, n)] = o
        o += ldims[m] * ldims[n]
    return offs


def exchange(local_blocks, dims, world: int, rank: int, dist, out):
    """Assemble the global blocks in `out` (torch tensor, global layout) from
    this rank's `local_blocks` (torch tensor, layout of its slab dims)."""
    import torch

    d = len(dims)
    lo, hi = slab_bounds(dims[-1], world, rank)
    ld = local_dims(dims, lo, hi)
    loffs = local_offsets(ld)
    maxs = max(slab_bounds(dims[-1], world, r)[1] - slab_bounds(dims[-1], world, r)[0]
               for r in range(world))
    reduce_parts = []
    for s in exchange_plan(dims):
        lo_off = loffs[(s.m, s.n)]
        if not s.gathered:
            seg = out[s.offset:s.offset + s.rows * s.cols]
            seg.copy_(local_blocks[lo_off:lo_off + s.rows * s.cols])
            reduce_parts.append(seg)
        else:
            mine = local_blocks[lo_off:lo_off + s.rows * (hi - lo)]
            if world == 1:
                out[s.offset:s.offset + s.rows * s.cols].copy_(mine)
                continue
            padded = torch.zeros(s.rows * maxs, dtype=local_blocks.dtype, device=local_blocks.device)
            padded[:mine.numel()].copy_(mine)
            gathered = torch.empty(world * s.rows * maxs, dtype=local_blocks.dtype,
                                   device=local_blocks.device)
            dist.all_gather_into_tensor(gathered, padded)
            for r in range(world):
                rlo, rhi = slab_bounds(dims[-1], world, r)
                dst = out[s.offset + s.rows * rlo:s.offset + s.rows * rhi]
                dst.copy_(gathered[r * s.rows * maxs:r * s.rows * maxs + s.rows * (rhi - rlo)])
    if world > 1 and reduce_parts:
        # one flat all-reduce over the (contiguous) partial blocks: they are the
        # pairs with n < d-1, which precede every (m, d-1) pair of the same row,
        # so reduce them one by one (few, and the block set is small)
        for seg in reduce_parts:
            dist.all_reduce(seg)
    return out


def exchange_numpy(local_list, dims):
    """Reference assembly without a process group (tests): local_list[r] is
    rank r's local block buffer."""
    world = len(local_list)
    total = sum(dims[m] * dims[n] for m, n in pairs(len(dims)))
    out = np.zeros(total)
    for s in exchange_plan(dims):
        seg = out[s.offset:s.offset + s.rows * s.cols]
        for r in range(world):
            lo, hi = slab_bounds(dims[-1], world, r)
            lo_off = local_offsets(local_dims(dims, lo, hi))[(s.m, s.n)]
            if s.gathered:
                seg[s.rows * lo:s.rows * hi] = local_list[r][lo_off:lo_off + s.rows * (hi - lo)]
            else:
                seg += local_list[r][lo_off:lo_off + s.rows * s.cols]
    return out
