"""B200-native HOSCF / iHOSCF best rank-one approximation (arXiv 2403.01778).

Python host mirror of the reference's C++ API (proj/include/rank1/*.hpp):
same names, argument meaning, defaults and error behaviour, every call going
through the C-ABI of librank1_b200.so (include/rank1_b200.h) into sm_100a
kernels.  There is no CPU fallback: without a B200 the calls raise
`DeviceError`.

Layout is the reference's: a DenseTensor is column-major (first index fastest,
tensor.hpp:11-14), blocks of J are column-major I_m x I_n (matrix.hpp:10).

    invalid_argument  -> InvalidArgument (a ValueError)
    runtime_error     -> Rank1RuntimeError (a RuntimeError)
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _lib
from ._lib import (DeviceError, InvalidArgument, Rank1Error, Rank1RuntimeError, check, dims_arr,
                   dptr, lib, u64p)

__all__ = [
    "DenseTensor", "FactorSet", "BuildOptions", "SymBlockMatrix", "KktReport", "EigPair",
    "SolveOptions", "IterationRecord", "SolveReport", "StackedVector", "SplitResult",
    "build_j", "build_j_serial", "build_block", "kkt_report", "scf_stopping_value",
    "largest_magnitude_eigenpair", "rayleigh_quotient_step", "split_factors", "stack_factors",
    "hoscf", "ihoscf", "solve", "solver_names", "Context", "DeviceTensor", "default_context",
    "InvalidArgument", "Rank1RuntimeError", "DeviceError", "Rank1Error",
]


# ------------------------------------------------------------- context --

class Context:
    """Owns a device, a stream and the workspaces (r1_context)."""

    def __init__(self, device: int = 0):
        h = ctypes.c_void_p()
        check(lib().r1_context_create(device, ctypes.byref(h)))
        self.handle = h
        self.device = device

    def close(self):
        if self.handle:
            lib().r1_context_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream_ptr: Optional[int]):
        check(lib().r1_context_set_stream(self.handle, ctypes.c_void_p(stream_ptr or 0)))
        self.stream_ptr = stream_ptr or 0

    def synchronize(self):
        check(lib().r1_context_synchronize(self.handle))

    @property
    def launch_count(self) -> int:
        v = ctypes.c_uint64()
        check(lib().r1_context_launch_count(self.handle, ctypes.byref(v)))
        return int(v.value)

    def sweep_plan_info(self, dims) -> dict:
        info = (ctypes.c_int64 * 16)()
        d = dims_arr(dims)
        check(lib().r1x_sweep_plan_info(self.handle, u64p(d), len(dims), info))
        keys = ["r0", "t1", "G0", "G1", "ncta", "nseg", "levels", "work_elems", "smem", "nra", "K", "KO",
                "ndyn", "ns", "ts"]
        return dict(zip(keys, [int(v) for v in info]))


_default: Optional[Context] = None


def default_context() -> Context:
    global _default
    if _default is None:
        _default = Context(0)
    return _default


class DeviceTensor:
    """A dense tensor resident in HBM (r1_tensor)."""

    def __init__(self, ctx: Context, handle, dims, keepalive=None):
        self.ctx = ctx
        self.handle = handle
        self.dims = tuple(int(d) for d in dims)
        self._keep = keepalive

    @classmethod
    def from_host(cls, data: np.ndarray, dims, ctx: Optional[Context] = None):
        ctx = ctx or default_context()
        a = np.ascontiguousarray(np.asarray(data, dtype=np.float64).reshape(-1))
        d = dims_arr(dims)
        if a.size != int(np.prod(d)):
            raise InvalidArgument("DenseTensor: data length does not match product of dims")
        h = ctypes.c_void_p()
        check(lib().r1_tensor_from_host(ctx.handle, dptr(a), u64p(d), len(dims), ctypes.byref(h)))
        return cls(ctx, h, dims)

    @classmethod
    def wrap(cls, dev_ptr: int, dims, ctx: Optional[Context] = None, keepalive=None):
        ctx = ctx or default_context()
        d = dims_arr(dims)
        h = ctypes.c_void_p()
        check(lib().r1_tensor_wrap_device(ctx.handle, ctypes.c_void_p(dev_ptr), u64p(d), len(dims),
                                          ctypes.byref(h)))
        return cls(ctx, h, dims, keepalive)

    @property
    def ptr(self) -> int:
        return int(lib().r1_tensor_device_ptr(self.handle) or 0)

    def copy_from_host(self, data: np.ndarray):
        a = np.ascontiguousarray(np.asarray(data, dtype=np.float64).reshape(-1))
        check(lib().r1_tensor_copy_from_host(self.ctx.handle, self.handle, dptr(a)))

    def to_host(self) -> np.ndarray:
        out = np.empty(int(np.prod(self.dims)))
        check(lib().r1_tensor_copy_to_host(self.ctx.handle, self.handle, dptr(out)))
        return out

    @classmethod
    def read_dt1(cls, path, ctx: Optional[Context] = None) -> "DeviceTensor":
        """read_dt1 (tensor_io.cpp:66-100) straight into HBM."""
        ctx = ctx or default_context()
        h = ctypes.c_void_p()
        check(lib().r1_tensor_read_dt1(ctx.handle, str(path).encode(), ctypes.byref(h)))
        # the header was validated by the loader; re-read its dims for the wrapper
        with open(path, "rb") as f:
            f.read(6)
            d = f.read(1)[0]
            dims = [int.from_bytes(f.read(8), "little") for _ in range(d)]
        return cls(ctx, h, dims)

    def write_dt1(self, path):
        """write_dt1 (tensor_io.cpp:47-64) straight from HBM."""
        check(lib().r1_tensor_write_dt1(self.ctx.handle, self.handle, str(path).encode()))

    def close(self):
        if self.handle:
            lib().r1_tensor_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ----------------------------------------------------------------- types --

class DenseTensor:
    """Column-major dense tensor (tensor.hpp:15-41)."""

    def __init__(self, dims: Sequence[int], data: Optional[np.ndarray] = None):
        dims = [int(d) for d in dims]
        if len(dims) == 0:
            raise InvalidArgument("DenseTensor: order must be >= 1")
        if any(d == 0 for d in dims):
            raise InvalidArgument("DenseTensor: all dims must be >= 1")
        n = int(np.prod(dims))
        if data is None:
            data = np.zeros(n)
        data = np.ascontiguousarray(np.asarray(data, dtype=np.float64).reshape(-1))
        if data.size != n:
            raise InvalidArgument("DenseTensor: data length does not match product of dims")
        self._dims = tuple(dims)
        self.data = data

    def order(self) -> int:
        return len(self._dims)

    def dim(self, n: int) -> int:
        return self._dims[n]

    def dims(self):
        return list(self._dims)

    def size(self) -> int:
        return self.data.size

    def values(self) -> np.ndarray:
        return self.data


@dataclass
class FactorSet:
    """lambda * u(0) o ... o u(d-1) (tensor.hpp:44-49)."""
    lambda_: float = 0.0
    factors: list = field(default_factory=list)

    def order(self) -> int:
        return len(self.factors)


@dataclass
class BuildOptions:
    """nepv.hpp:45-49.  The device sweep is deterministic for any setting."""
    threads: int = 0
    determinism: bool = True
    reuse_intermediates: bool = False


class SymBlockMatrix:
    """J = scale * [B(m,n)] kept as its upper blocks (nepv.hpp:15-43)."""

    def __init__(self, block_dims, blocks: Optional[np.ndarray] = None):
        self._dims = [int(d) for d in block_dims]
        d = len(self._dims)
        if d < 2:
            raise InvalidArgument("SymBlockMatrix: order must be >= 2")
        n = sum(self._dims[m] * self._dims[k] for m in range(d) for k in range(m + 1, d))
        self.blocks = np.zeros(n) if blocks is None else np.ascontiguousarray(blocks, dtype=np.float64)
        self._scale = 1.0 / (d - 1)
        self._offs = {}
        o = 0
        for m in range(d):
            for k in range(m + 1, d):
                self._offs[(m, k)] = o
                o += self._dims[m] * self._dims[k]

    def order(self) -> int:
        return len(self._dims)

    def total_dim(self) -> int:
        return sum(self._dims)

    def block_dims(self):
        return list(self._dims)

    def scale(self) -> float:
        return self._scale

    def block(self, m: int, n: int) -> np.ndarray:
        if m >= n or n >= len(self._dims):
            raise InvalidArgument("SymBlockMatrix: bad block pair")
        o = self._offs[(m, n)]
        return self.blocks[o:o + self._dims[m] * self._dims[n]].reshape(
            self._dims[m], self._dims[n], order="F")

    def matvec(self, x) -> np.ndarray:
        x = np.asarray(x, dtype=np.float64)
        if x.size != self.total_dim():
            raise InvalidArgument("SymBlockMatrix: matvec size mismatch")
        off = np.concatenate([[0], np.cumsum(self._dims)]).astype(int)
        y = np.zeros(off[-1])
        d = len(self._dims)
        for m in range(d):
            for k in range(m + 1, d):
                b = self.block(m, k)
                y[off[m]:off[m + 1]] += b @ x[off[k]:off[k + 1]]
                y[off[k]:off[k + 1]] += b.T @ x[off[m]:off[m + 1]]
        return y * self._scale

    def dense(self) -> np.ndarray:
        off = np.concatenate([[0], np.cumsum(self._dims)]).astype(int)
        s = np.zeros((off[-1], off[-1]))
        d = len(self._dims)
        for m in range(d):
            for k in range(m + 1, d):
                b = self.block(m, k) * self._scale
                s[off[m]:off[m + 1], off[k]:off[k + 1]] = b
                s[off[k]:off[k + 1], off[m]:off[m + 1]] = b.T
        return s

    def frobenius_norm(self) -> float:
        return math.sqrt(2.0 * float(np.dot(self.blocks, self.blocks))) * self._scale


@dataclass
class KktReport:
    lambda_: float = 0.0
    per_mode_residuals: list = field(default_factory=list)
    max_residual: float = 0.0


@dataclass
class EigPair:
    value: float = 0.0
    vector: np.ndarray = field(default_factory=lambda: np.zeros(0))


class StackedVector:
    """stacked.hpp:13-38."""

    def __init__(self, block_dims, flat: Optional[np.ndarray] = None):
        self._dims = [int(d) for d in block_dims]
        n = sum(self._dims)
        if flat is None:
            flat = np.zeros(n)
        flat = np.ascontiguousarray(np.asarray(flat, dtype=np.float64))
        if flat.size != n:
            raise InvalidArgument("StackedVector: flat length does not match block dims")
        self._flat = flat
        self._offs = np.concatenate([[0], np.cumsum(self._dims)]).astype(int)

    def order(self):
        return len(self._dims)

    def total_dim(self):
        return self._flat.size

    def block_dims(self):
        return list(self._dims)

    def block(self, n: int) -> np.ndarray:
        return self._flat[self._offs[n]:self._offs[n + 1]]

    def flat(self) -> np.ndarray:
        return self._flat

    def block_norm(self, n: int) -> float:
        return float(np.linalg.norm(self.block(n)))

    def norm(self) -> float:
        return float(np.linalg.norm(self._flat))


@dataclass
class SplitResult:
    factors: FactorSet
    degenerate: list

    def any_degenerate(self) -> bool:
        return any(self.degenerate)


def _norm2_seq(v) -> float:
    s = 0.0
    for x in np.asarray(v, dtype=np.float64).tolist():
        s += x * x
    return math.sqrt(s)


def split_factors(x: StackedVector) -> SplitResult:
    """stacked.cpp:40-58 (host-side; the solver runs the device version)."""
    fs, deg = [], []
    for n in range(x.order()):
        blk = np.array(x.block(n))
        nrm = _norm2_seq(blk)
        if nrm < 1e-12:
            fs.append(np.zeros_like(blk))
            deg.append(1)
        else:
            fs.append(blk / nrm)
            deg.append(0)
    return SplitResult(FactorSet(0.0, fs), deg)


def stack_factors(f: FactorSet) -> StackedVector:
    """stacked.cpp:60-73."""
    if f.order() == 0:
        raise InvalidArgument("stack_factors: empty factor set")
    if max(abs(_norm2_seq(u) - 1.0) for u in f.factors) > 1e-8:
        raise InvalidArgument("stack_factors: factors must have unit norm")
    s = 1.0 / math.sqrt(f.order())
    return StackedVector([len(u) for u in f.factors],
                         np.concatenate([np.asarray(u, dtype=np.float64) * s for u in f.factors]))


@dataclass
class SolveOptions:
    """solvers.hpp:17-31 (same defaults) + two device-side stop extensions:
    scf_lambda_rtol (relative sigma change) and scf_angle_tol (factor change,
    |sin angle(x_k, x_{k-1})|); 0 = off."""
    tol: float = 1e-4
    max_iters: int = 500
    seed: int = 0
    init: str = "uniform01"          # "uniform01" | "provided"
    init_factors: list = field(default_factory=list)
    determinism: bool = True
    rqi_accept_rule: str = "magnitude"  # "magnitude" | "signed_increase"
    stop_rule: str = "kkt"
    threads: int = 0
    record_kkt: bool = True
    asvd_disjoint_pairs: bool = False
    reuse_intermediates: bool = False
    scf_lambda_rtol: float = 0.0
    scf_angle_tol: float = 0.0


@dataclass
class IterationRecord:
    lambda_: float = 0.0
    stop_value: float = 0.0
    eq11_value: float = 0.0
    kkt_max_residual: float = 0.0
    rqi_accepted: bool = False
    lambda_pre_rqi: float = 0.0
    t_build_j: float = 0.0
    t_eig: float = 0.0
    t_other: float = 0.0
    n_sweeps: int = 1
    factor_change: float = -1.0


@dataclass
class SolveReport:
    algorithm: str = ""
    result: FactorSet = field(default_factory=FactorSet)
    converged: bool = False
    iterations: int = 0
    lambda0: float = 0.0
    restarted: bool = False
    trace: list = field(default_factory=list)
    final_x: Optional[StackedVector] = None
    total_sweeps: int = 0
    t_total: float = 0.0

    def wall_build_j(self) -> float:
        return sum(r.t_build_j for r in self.trace)

    def wall_eig(self) -> float:
        return sum(r.t_eig for r in self.trace)

    def wall_total(self) -> float:
        return sum(r.t_build_j + r.t_eig + r.t_other for r in self.trace)


# ------------------------------------------------------------ the sweep --

def _check_factor_shapes(a: DenseTensor, f: FactorSet):
    """nepv.cpp:24-29."""
    if f.order() != a.order():
        raise InvalidArgument("factor set order mismatch")
    for k in range(a.order()):
        if len(f.factors[k]) != a.dim(k):
            raise InvalidArgument("factor length does not match tensor dim")


def _flat(f: FactorSet) -> np.ndarray:
    return np.ascontiguousarray(np.concatenate([np.asarray(u, dtype=np.float64).reshape(-1)
                                                for u in f.factors]))


def _tensor_args(a):
    if isinstance(a, DeviceTensor):
        return None, a.handle, a.dims
    return a.data, None, a.dims()


def build_j(a, f: FactorSet, opts: BuildOptions = BuildOptions(), ctx: Optional[Context] = None
            ) -> SymBlockMatrix:
    """All P = d(d-1)/2 blocks of J(u) on the device (nepv.hpp:58).  `a` may be a
    host DenseTensor (copied to HBM per call) or a resident DeviceTensor."""
    ctx = ctx or default_context()
    host, dev, dims = _tensor_args(a)
    if len(dims) < 2:
        raise InvalidArgument("build_j: tensor order must be >= 2")
    if isinstance(a, DenseTensor):
        _check_factor_shapes(a, f)
    fl = _flat(f)
    d = dims_arr(dims)
    out = SymBlockMatrix(dims)
    hp = dptr(host) if host is not None else None
    check(lib().r1_build_j(ctx.handle, hp, dev, u64p(d), len(dims), dptr(fl), dptr(out.blocks)))
    return out


def build_j_serial(a, f: FactorSet, ctx: Optional[Context] = None) -> SymBlockMatrix:
    """nepv.hpp:62 — the same deterministic device path."""
    if a.order() < 2 if isinstance(a, DenseTensor) else len(a.dims) < 2:
        raise InvalidArgument("build_j_serial: tensor order must be >= 2")
    return build_j(a, f, BuildOptions(), ctx)


def build_block(a, f: FactorSet, m: int, n: int, ctx: Optional[Context] = None) -> np.ndarray:
    """nepv.hpp:54: block (m,n) as an I_m x I_n array (rows = lower mode)."""
    ctx = ctx or default_context()
    host, dev, dims = _tensor_args(a)
    if len(dims) < 2:
        raise InvalidArgument("build_block: tensor order must be >= 2")
    if m == n:
        raise InvalidArgument("build_block: block modes must differ")
    if m > n:
        m, n = n, m
    if n >= len(dims):
        raise InvalidArgument("build_block: mode out of range")
    if isinstance(a, DenseTensor):
        _check_factor_shapes(a, f)
    fl = _flat(f)
    d = dims_arr(dims)
    out = np.empty(dims[m] * dims[n])
    hp = dptr(host) if host is not None else None
    check(lib().r1_build_block(ctx.handle, hp, dev, u64p(d), len(dims), dptr(fl), m, n, dptr(out)))
    return out.reshape(dims[m], dims[n], order="F")


def kkt_report(a, f: FactorSet, parallel: bool = False, ctx: Optional[Context] = None
               ) -> KktReport:
    """nepv.hpp:72 — one device sweep plus the block identities
    w_n = B(n,m) u_m and lambda = u_0' B(0,1) u_1 (no extra tensor passes)."""
    ctx = ctx or default_context()
    host, dev, dims = _tensor_args(a)
    if isinstance(a, DenseTensor):
        _check_factor_shapes(a, f)
    fl = _flat(f)
    d = dims_arr(dims)
    out = np.empty(len(dims) + 2)
    hp = dptr(host) if host is not None else None
    check(lib().r1_kkt_report(ctx.handle, hp, dev, u64p(d), len(dims), dptr(fl), dptr(out)))
    return KktReport(float(out[0]), [float(v) for v in out[2:]], float(out[1]))


def scf_stopping_value(j: SymBlockMatrix, x: StackedVector, lam: float,
                       ctx: Optional[Context] = None) -> float:
    """Eq. 11 (nepv.hpp:77) on the device."""
    ctx = ctx or default_context()
    if x.total_dim() != j.total_dim():
        raise InvalidArgument("scf_stopping_value: dimension mismatch")
    d = dims_arr(j.block_dims())
    out = ctypes.c_double()
    xf = np.ascontiguousarray(x.flat())
    check(lib().r1_scf_stopping_value(ctx.handle, u64p(d), j.order(), dptr(j.blocks), dptr(xf),
                                      float(lam), ctypes.byref(out)))
    return out.value


def largest_magnitude_eigenpair(s: np.ndarray, ctx: Optional[Context] = None) -> EigPair:
    """sym_eig.hpp:30 on the device (Lanczos, both spectral ends)."""
    ctx = ctx or default_context()
    s = np.asarray(s, dtype=np.float64)
    if s.ndim != 2 or s.shape[0] != s.shape[1]:
        raise InvalidArgument("sym_eig: matrix must be square")
    n = s.shape[0]
    if n == 0:
        raise InvalidArgument("largest_magnitude_eigenpair: empty matrix")
    sf = np.ascontiguousarray(s.reshape(-1, order="F"))
    val = ctypes.c_double()
    vec = np.empty(n)
    check(lib().r1_largest_magnitude_eigenpair(ctx.handle, n, dptr(sf), ctypes.byref(val),
                                               dptr(vec)))
    return EigPair(val.value, vec)


def eig_blocks(j: SymBlockMatrix, ctx: Optional[Context] = None):
    """Largest-magnitude eigenpair of the block matrix J on the device (the
    solver's eigen step).  Returns (EigPair, info dict)."""
    ctx = ctx or default_context()
    d = dims_arr(j.block_dims())
    n = j.total_dim()
    val = ctypes.c_double()
    vec = np.empty(n)
    info = (ctypes.c_int * 5)()
    stats = np.zeros(5)
    check(lib().r1x_eig_blocks_info(ctx.handle, u64p(d), j.order(), dptr(j.blocks),
                                    ctypes.byref(val), dptr(vec), info, dptr(stats)))
    keys = ["converged", "pick", "steps", "restarts", "breakdowns"]
    inf = dict(zip(keys, [int(v) for v in info]))
    inf.update(theta_lo=stats[0], theta_hi=stats[1], res_lo=stats[2], res_hi=stats[3])
    return EigPair(val.value, vec), inf


def rayleigh_quotient_step(s: np.ndarray, x, ctx: Optional[Context] = None):
    """sym_eig.hpp:37-38 on the device; None reproduces std::nullopt."""
    ctx = ctx or default_context()
    s = np.asarray(s, dtype=np.float64)
    x = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    n = s.shape[0]
    if s.ndim != 2 or s.shape[1] != n or x.size != n:
        raise InvalidArgument("rayleigh_quotient_step: size mismatch")
    sf = np.ascontiguousarray(s.reshape(-1, order="F"))
    y = np.empty(n)
    acc = ctypes.c_int()
    check(lib().r1_rayleigh_quotient_step(ctx.handle, n, dptr(sf), dptr(x), dptr(y),
                                          ctypes.byref(acc)))
    return y if acc.value else None


# ---------------------------------------------------------------- solvers --

_SOLVERS = ["hoscf", "ihoscf", "hopm", "jacobi_hopm", "asvd", "jacobi_asvd"]


def solver_names():
    return list(_SOLVERS)


def _options_c(o: SolveOptions, dims):
    c = _lib.SolveOptionsC()
    lib().r1_solve_options_default(ctypes.byref(c))
    c.tol = o.tol
    c.max_iters = o.max_iters
    c.seed = o.seed
    c.determinism = 1 if o.determinism else 0
    c.rqi_accept_rule = 1 if o.rqi_accept_rule == "signed_increase" else 0
    c.stop_rule = {"kkt": 0, "eq11": 1, "lambda_delta": 2}[o.stop_rule]
    c.threads = o.threads
    c.record_kkt = 1 if o.record_kkt else 0
    c.reuse_intermediates = 1 if o.reuse_intermediates else 0
    c.asvd_disjoint_pairs = 1 if o.asvd_disjoint_pairs else 0
    c.scf_lambda_rtol = o.scf_lambda_rtol
    c.scf_angle_tol = o.scf_angle_tol
    keep = None
    if o.init == "provided":
        if len(o.init_factors) != len(dims):
            raise InvalidArgument("solver: provided init has wrong order")
        for k, u in enumerate(o.init_factors):
            if len(u) != dims[k]:
                raise InvalidArgument("solver: provided init factor length mismatch")
        keep = np.ascontiguousarray(np.concatenate([np.asarray(u, dtype=np.float64)
                                                    for u in o.init_factors]))
        c.init = 1
        c.init_factors = dptr(keep)
    return c, keep


def solve(algorithm: str, a, opts: SolveOptions, ctx: Optional[Context] = None,
          global_dims=None) -> SolveReport:
    """solvers.hpp:86: every solver of the reference on the device —
    hoscf | ihoscf (SCF on J(u)) and the baselines hopm | jacobi_hopm | asvd |
    jacobi_asvd (solvers.cpp:299-447) on the same device sweep.

    global_dims: `a` is this rank's slab of a tensor sharded along its last mode
    (r1_solve_sharded; the context needs a communicator, distributed.init_comm)."""
    ctx = ctx or default_context()
    if algorithm not in _SOLVERS:
        raise InvalidArgument("unknown solver: " + algorithm)
    owned = None
    if isinstance(a, DenseTensor):
        if a.order() < 2:
            raise InvalidArgument("solver: tensor order must be >= 2")
        owned = DeviceTensor.from_host(a.data, a.dims(), ctx)
        t = owned
    else:
        t = a
    dims = list(t.dims) if global_dims is None else [int(v) for v in global_dims]
    c, keep = _options_c(opts, dims)
    n = sum(dims)
    fac = np.empty(n)
    fx = np.empty(n)
    tr = (_lib.IterationRecordC * max(1, opts.max_iters))()
    r = _lib.SolveReportC()
    r.factors = dptr(fac)
    r.final_x = dptr(fx)
    r.trace = tr
    try:
        if global_dims is None:
            check(lib().r1_solve(ctx.handle, algorithm.encode(), t.handle, ctypes.byref(c),
                                 ctypes.byref(r)))
        else:
            gd = _lib.dims_arr(dims)
            check(lib().r1_solve_sharded(ctx.handle, algorithm.encode(), t.handle, _lib.u64p(gd),
                                         len(dims), ctypes.byref(c), ctypes.byref(r)))
    finally:
        if owned is not None:
            owned.close()
    offs = np.concatenate([[0], np.cumsum(dims)]).astype(int)
    rep = SolveReport(algorithm=algorithm)
    rep.result = FactorSet(r.lambda_, [fac[offs[k]:offs[k + 1]].copy() for k in range(len(dims))])
    rep.converged = bool(r.converged)
    rep.iterations = int(r.iterations)
    rep.lambda0 = r.lambda0
    rep.restarted = bool(r.restarted)
    # SCF solvers: last stacked eigenvector; baselines: empty (solvers.hpp:56)
    rep.final_x = StackedVector(dims, fx.copy()) if algorithm in ("hoscf", "ihoscf") else None
    rep.total_sweeps = int(r.total_sweeps)
    rep.t_total = r.t_total
    for i in range(rep.iterations):
        t_ = tr[i]
        rep.trace.append(IterationRecord(t_.lambda_, t_.stop_value, t_.eq11_value,
                                         t_.kkt_max_residual, bool(t_.rqi_accepted),
                                         t_.lambda_pre_rqi, t_.t_build_j, t_.t_eig, t_.t_other,
                                         int(t_.n_sweeps), t_.factor_change))
    return rep


def hoscf(a, opts: SolveOptions, ctx: Optional[Context] = None) -> SolveReport:
    """solvers.hpp:63."""
    return solve("hoscf", a, opts, ctx)


def ihoscf(a, opts: SolveOptions, ctx: Optional[Context] = None) -> SolveReport:
    """solvers.hpp:68."""
    return solve("ihoscf", a, opts, ctx)


def hopm(a, opts: SolveOptions, ctx: Optional[Context] = None) -> SolveReport:
    """solvers.hpp:70-72: Gauss-Seidel power sweep (ALS)."""
    return solve("hopm", a, opts, ctx)


def jacobi_hopm(a, opts: SolveOptions, ctx: Optional[Context] = None) -> SolveReport:
    """solvers.hpp:74-76: power sweep in Jacobi form."""
    return solve("jacobi_hopm", a, opts, ctx)


def asvd(a, opts: SolveOptions, ctx: Optional[Context] = None) -> SolveReport:
    """solvers.hpp:78-80: alternating SVD over adjacent mode pairs."""
    return solve("asvd", a, opts, ctx)


def jacobi_asvd(a, opts: SolveOptions, ctx: Optional[Context] = None) -> SolveReport:
    """solvers.hpp:82-83: asvd with all pair subproblems from the previous iterate."""
    return solve("jacobi_asvd", a, opts, ctx)


# ------------------------------------------------------- greedy deflation --

@dataclass
class GreedyReport:
    """greedy.hpp:11-17."""
    terms: list = field(default_factory=list)            # FactorSet per term
    residual_ratios: list = field(default_factory=list)  # ||R||_F / ||A||_F after each term
    solves: list = field(default_factory=list)           # SolveReport per term
    completed: bool = False
    failure: str = ""


def greedy_rank_r(a, r: int, solver: str, opts: SolveOptions,
                  ctx: Optional[Context] = None) -> GreedyReport:
    """greedy_rank_r (greedy.hpp:21-22, greedy.cpp:7-35) with the residual kept in
    HBM: per term a device solve (seed + term) and one fused subtract + norm pass."""
    ctx = ctx or default_context()
    if r < 1:
        raise InvalidArgument("greedy_rank_r: rank must be >= 1")
    owned = None
    if isinstance(a, DenseTensor):
        owned = DeviceTensor.from_host(a.data, a.dims(), ctx)
        t = owned
    else:
        t = a
    dims = list(t.dims)
    n = sum(dims)
    c, keep = _options_c(opts, dims)
    lam = np.zeros(r)
    fac = np.zeros(r * n)
    rat = np.zeros(r)
    solves = (_lib.SolveReportC * r)()
    bufs = []
    for i in range(r):
        f_, x_ = np.empty(n), np.empty(n)
        tr = (_lib.IterationRecordC * max(1, opts.max_iters))()
        bufs.append((f_, x_, tr))
        solves[i].factors = dptr(f_)
        solves[i].final_x = dptr(x_)
        solves[i].trace = tr
    g = _lib.GreedyReportC()
    g.lambdas, g.factors, g.residual_ratios = dptr(lam), dptr(fac), dptr(rat)
    g.solves = solves
    try:
        check(lib().r1_greedy_rank_r(ctx.handle, t.handle, ctypes.c_uint64(r), solver.encode(),
                                     ctypes.byref(c), ctypes.byref(g)))
    finally:
        if owned is not None:
            owned.close()
    offs = np.concatenate([[0], np.cumsum(dims)]).astype(int)
    rep = GreedyReport(completed=bool(g.completed), failure=g.failure.decode())
    for i in range(g.terms):
        rep.terms.append(FactorSet(lam[i], [fac[i * n + offs[k]:i * n + offs[k + 1]].copy()
                                            for k in range(len(dims))]))
        rep.residual_ratios.append(float(rat[i]))
        s_ = solves[i]
        sr = SolveReport(algorithm=solver)
        sr.result = rep.terms[-1]
        sr.converged, sr.iterations = bool(s_.converged), int(s_.iterations)
        sr.lambda0, sr.restarted = s_.lambda0, bool(s_.restarted)
        sr.total_sweeps = int(s_.total_sweeps)
        rep.solves.append(sr)
    return rep


def read_dt1(path, ctx: Optional[Context] = None) -> DeviceTensor:
    """tensor_io.hpp:17: a .dt1 file straight into HBM."""
    return DeviceTensor.read_dt1(path, ctx)


def write_dt1(path, a) -> None:
    """tensor_io.hpp:16: a DeviceTensor (from HBM) or a DenseTensor to a .dt1 file."""
    if isinstance(a, DeviceTensor):
        a.write_dt1(path)
        return
    t = DeviceTensor.from_host(a.data, a.dims())
    try:
        t.write_dt1(path)
    finally:
        t.close()
