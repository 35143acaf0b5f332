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
            if dims[-1] % world == 0:
                # even slabs: rank r's columns are the r-th chunk of the
                # column-major block, so NCCL gathers straight into place
                dist.all_gather_into_tensor(out[s.offset:s.offset + s.rows * s.cols], mine)
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


# ---------------------------------------------------------------------------
# Distributed HOSCF / iHOSCF: the tensor stays sharded in slabs;
# per sweep each rank contracts its slab on its GPU and exchange() assembles
# the replicated blocks of J; the eigen step, the RQI and the stopping test run
# replicated on every rank on identical bits (NCCL returns the same reduced
# values to every rank), so every rank takes the same branch.  The control
# flow is run_hoscf / run_ihoscf (solvers.cpp:129-297), as in csrc/solver.cu.

_G = 0x9E3779B97F4A7C15
_M = (1 << 64) - 1


def _mix(z):
    z ^= z >> 30
    z = (z * 0xBF58476D1CE4E5B9) & _M
    z ^= z >> 27
    z = (z * 0x94D049BB133111EB) & _M
    z ^= z >> 31
    return z


def random_unit_factors(dims, seed: int, stream: int):
    """random_unit_factors (solvers.cpp:34-49): CounterRng(seed, stream) uniform
    draws mode by mode, normalised (all-zero -> normalised ones)."""
    key = _mix((seed + _G * (stream + 1)) & _M)
    c = 0
    out = []
    for n in dims:
        u = np.empty(n)
        for i in range(n):
            c += 1
            u[i] = (_mix((key + _G * c) & _M) >> 11) * 2.0 ** -53
        s = 0.0
        for v in u.tolist():
            s += v * v
        if s == 0.0:
            u = np.ones(n)
            s = float(n)
        out.append(u / np.sqrt(s))
    return out


class _Degenerate(Exception):
    pass


def solve_distributed(algorithm, slab, dims, opts, dist=None, world: int = 1, rank: int = 0,
                      ctx=None):
    """hoscf | ihoscf on a tensor sharded in slabs along reference mode d-1.

    slab: this rank's DeviceTensor (dims[:-1] + [hi-lo]); dims: global dims.
    Returns the reference-shaped SolveReport (identical on every rank)."""
    import ctypes
    import time

    import torch

    from . import (DeviceTensor, FactorSet, InvalidArgument, IterationRecord, Rank1RuntimeError,
                   SolveReport, StackedVector, _lib, default_context)

    if algorithm not in ("hoscf", "ihoscf"):
        raise InvalidArgument("solve_distributed: hoscf | ihoscf")
    if len(dims) < 2:
        raise InvalidArgument("solver: tensor order must be >= 2")
    if not opts.tol > 0.0:
        raise InvalidArgument("solver: tol must be > 0")
    if opts.max_iters < 1:
        raise InvalidArgument("solver: max_iters must be >= 1")
    ctx = ctx or default_context()
    L = _lib.lib()
    dims = [int(v) for v in dims]
    d = len(dims)
    n = sum(dims)
    lo, hi = slab_bounds(dims[-1], world, rank)
    nb = sum(dims[m] * dims[k] for m, k in pairs(d))
    ld = local_dims(dims, lo, hi)
    nbl = sum(ld[m] * ld[k] for m, k in pairs(d))
    dev = torch.device("cuda", torch.cuda.current_device())
    f64 = dict(dtype=torch.float64, device=dev)
    fac = torch.empty(sum(ld), **f64)
    lblocks = torch.empty(max(nbl, 1), **f64)
    gJ = [torch.empty(nb, **f64), torch.empty(nb, **f64)]
    xv, yv, vec, val = (torch.empty(n, **f64), torch.empty(n, **f64), torch.empty(n, **f64),
                        torch.empty(1, **f64))
    gdims = _lib.dims_arr(dims)
    offs = np.concatenate([[0], np.cumsum(dims)]).astype(int)
    accelerated = algorithm == "ihoscf"
    stream = torch.cuda.current_stream()

    def sweep(u, out):
        fl = np.concatenate([np.asarray(v, dtype=np.float64) for v in u[:-1]] + [u[-1][lo:hi]])
        fac.copy_(torch.from_numpy(fl))
        _lib.check(L.r1_build_j_device(ctx.handle, slab.handle, ctypes.c_void_p(fac.data_ptr()),
                                       ctypes.c_void_p(lblocks.data_ptr()), None))
        if world > 1:
            exchange(lblocks[:nbl], dims, world, rank, dist, out)
        else:
            out.copy_(lblocks[:nb])

    def frob(J):
        t = DeviceTensor.wrap(J.data_ptr(), (nb, 1), ctx, keepalive=J)
        r = ctypes.c_double()
        _lib.check(L.r1_tensor_frobenius(ctx.handle, t.handle, ctypes.byref(r)))
        t.close()
        return r.value

    def matvec(J, x_host):
        xv.copy_(torch.from_numpy(np.ascontiguousarray(x_host)))
        _lib.check(L.r1_block_matvec_device(ctx.handle, _lib.u64p(gdims), d,
                                            ctypes.c_void_p(J.data_ptr()),
                                            ctypes.c_void_p(xv.data_ptr()),
                                            ctypes.c_void_p(yv.data_ptr())))
        return yv.cpu().numpy()

    def stack(u):
        return np.concatenate(u) / np.sqrt(d)

    def post(J, u, mu):
        """y = J xhat: rho, Eq. 11 (nepv.cpp:271-282), lambda = u_0'w_0, KKT."""
        xh = stack(u)
        y = matvec(J, xh)
        rho = float(np.dot(xh, y))
        fro = np.sqrt(2.0) * frob(J) / (d - 1)
        eq11 = float(np.linalg.norm(y - rho * xh)) / (fro + abs(mu))
        w = np.sqrt(d) * y
        lam = float(np.dot(u[0], w[offs[0]:offs[1]]))
        res = [float(np.linalg.norm(w[offs[k]:offs[k + 1]] - lam * u[k])) for k in range(d)]
        return rho, eq11, max(res), lam

    def split(x):
        u, deg = [], False
        for k in range(d):
            b = np.asarray(x[offs[k]:offs[k + 1]], dtype=np.float64)
            nrm = float(np.sqrt(np.dot(b, b)))
            if nrm < 1e-12:
                deg = True
                u.append(np.zeros_like(b))
            else:
                u.append(b / nrm)
        return u, deg

    def eig(J, x0):
        if x0 is not None:
            vec.copy_(torch.from_numpy(np.ascontiguousarray(x0)))
        _lib.check(L.r1_eig_blocks_device(ctx.handle, _lib.u64p(gdims), d,
                                          ctypes.c_void_p(J.data_ptr()),
                                          ctypes.c_void_p(vec.data_ptr()) if x0 is not None else None,
                                          ctypes.c_void_p(val.data_ptr()),
                                          ctypes.c_void_p(vec.data_ptr())))
        return float(val.item()), vec.cpu().numpy()

    def run(u):
        rep = SolveReport(algorithm=algorithm)
        cur, mid = 0, 1
        sweep(u, gJ[cur])
        rep.lambda0 = post(gJ[cur], u, 0.0)[3]
        sweeps = 1
        x_prev, lam_prev = None, None
        final_x = None
        for k in range(1, opts.max_iters + 1):
            t0 = time.perf_counter()
            mu, x = eig(gJ[cur], x_prev)
            t1 = time.perf_counter()
            u_mid, deg = split(x)
            if deg:
                raise _Degenerate()
            sweep(u_mid, gJ[mid])
            sweeps += 1
            torch.cuda.synchronize()
            t2 = time.perf_counter()
            rho_mid, sv, kkt_mid, _ = post(gJ[mid], u_mid, mu)
            rec = IterationRecord(lambda_=mu, lambda_pre_rqi=float("nan"), n_sweeps=1)
            xfinal = x
            if not accelerated or sv <= opts.tol:
                u, (cur, mid) = u_mid, (mid, cur)
                rec.eq11_value = rec.stop_value = sv
                rec.kkt_max_residual = kkt_mid if opts.record_kkt else float("nan")
            else:
                rec.lambda_pre_rqi = rho_mid
                accepted, rho_y = False, 0.0
                xv.copy_(torch.from_numpy(np.ascontiguousarray(stack(u_mid))))
                acc = ctypes.c_int()
                _lib.check(L.r1_rqi_blocks_device(ctx.handle, _lib.u64p(gdims), d,
                                                  ctypes.c_void_p(gJ[mid].data_ptr()),
                                                  ctypes.c_void_p(xv.data_ptr()),
                                                  ctypes.c_void_p(vec.data_ptr()), ctypes.byref(acc)))
                if acc.value:
                    yr = vec.cpu().numpy()
                    u_r, deg_r = split(yr)
                    if not deg_r:
                        rho_y = float(np.dot(yr, matvec(gJ[mid], yr)))
                        better = (rho_y > rho_mid) if opts.rqi_accept_rule == "signed_increase" \
                            else abs(rho_y) > abs(rho_mid)
                        accepted = better
                rec.rqi_accepted = accepted
                if accepted:
                    u = u_r
                    sweep(u, gJ[cur])
                    sweeps += 1
                    rec.n_sweeps += 1
                    _, eq, kk, _ = post(gJ[cur], u, rho_y)
                    rec.lambda_ = rho_y
                    rec.eq11_value = rec.stop_value = eq
                    rec.kkt_max_residual = kk if opts.record_kkt else float("nan")
                    xfinal = yr
                else:
                    u, (cur, mid) = u_mid, (mid, cur)
                    rec.lambda_ = rho_mid
                    rec.eq11_value = rec.stop_value = sv
                    rec.kkt_max_residual = kkt_mid if opts.record_kkt else float("nan")
            t3 = time.perf_counter()
            rec.t_eig, rec.t_build_j, rec.t_other = t1 - t0, t2 - t1, t3 - t2
            rep.trace.append(rec)
            rep.iterations = k
            x_prev = final_x = np.asarray(xfinal)
            if rec.stop_value <= opts.tol:
                rep.converged = True
                break
            if opts.scf_lambda_rtol > 0 and lam_prev is not None and \
                    abs(rec.lambda_ - lam_prev) <= opts.scf_lambda_rtol * abs(rec.lambda_):
                rep.converged = True
                break
            lam_prev = rec.lambda_
        lam = post(gJ[cur], u, 0.0)[3]
        if lam < 0:
            lam = -lam
            u = [-u[0]] + list(u[1:])
        rep.result = FactorSet(lam, [np.asarray(v).copy() for v in u])
        rep.final_x = StackedVector(dims, final_x) if final_x is not None else None
        rep.total_sweeps = sweeps
        return rep

    if opts.init == "provided":
        u0 = []
        for k, v in enumerate(opts.init_factors):
            v = np.asarray(v, dtype=np.float64)
            nrm = float(np.sqrt(np.dot(v, v)))
            if nrm == 0.0:
                raise InvalidArgument("solver: provided init factor is zero")
            u0.append(v / nrm)
    else:
        u0 = random_unit_factors(dims, opts.seed, 2)
    # the library's kernels and the torch copies / NCCL calls share one stream
    # (a dedicated one: handle 0, torch's legacy default stream, would select
    # the library's own stream)
    prev_stream = getattr(ctx, "stream_ptr", 0)
    work = stream if stream.cuda_stream else torch.cuda.Stream()
    work.wait_stream(torch.cuda.current_stream())
    t_start = time.perf_counter()
    try:
        with torch.cuda.stream(work):
            ctx.set_stream(work.cuda_stream)
            try:
                rep = run(u0)
            except _Degenerate:
                try:
                    rep = run(random_unit_factors(dims, opts.seed, 3))
                    rep.restarted = True
                except _Degenerate as e:
                    raise Rank1RuntimeError("solver failed after restart") from e
    finally:
        ctx.set_stream(prev_stream)
        torch.cuda.current_stream().wait_stream(work)
    rep.t_total = time.perf_counter() - t_start
    return rep
