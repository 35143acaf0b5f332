"""ORACLE / TEST INFRASTRUCTURE — CPU restatement of the reference hot path.

This module is the CHECKER for the CUDA path.  It is used only by tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline leg; the product package
never imports it.  Functions cite the reference (paths relative to
/root/reference/proj).  Parity of this restatement with the compiled reference
and with the reference's own known-answer tests is pinned in
tests/test_oracle_pins.py and tests/golden/.

Tensors are 1-D float64 arrays in the reference's column-major layout (first
index fastest, tensor.hpp:11-14) plus a `dims` tuple; factor sets are lists of
1-D arrays; J is the flat concatenation of its upper blocks in pair order
(nepv.cpp:98-102), each block column-major.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "librank1_oracle.so")
_lib = None

_dp = ctypes.POINTER(ctypes.c_double)
_u64p = ctypes.POINTER(ctypes.c_uint64)
_ip = ctypes.POINTER(ctypes.c_int)


def build() -> str:
    """Compile the C core (make -C oracle); cheap and idempotent."""
    subprocess.run(["make", "-s", "-C", _HERE, "_build/librank1_oracle.so"], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        L.r1o_rng_key.restype = ctypes.c_uint64
        L.r1o_rng_key.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
        for name in ("r1o_rng_units", "r1o_rng_gauss"):
            getattr(L, name).argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                         ctypes.c_int64, _dp]
        L.r1o_rng_u64.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                  ctypes.c_int64, _u64p]
        L.r1o_gen_gaussian.argtypes = [ctypes.c_uint64, ctypes.c_uint64, _dp]
        L.r1o_planted_factor.argtypes = [ctypes.c_uint64, ctypes.c_int, ctypes.c_int64, _dp]
        L.r1o_sumsq_blocked.restype = ctypes.c_double
        L.r1o_sumsq_blocked.argtypes = [_dp, ctypes.c_uint64]
        L.r1o_gen_config.restype = ctypes.c_int
        L.r1o_gen_config.argtypes = [ctypes.c_int, _u64p, ctypes.c_int, ctypes.c_uint64, _dp]
        L.r1o_block.argtypes = [_dp, _u64p, ctypes.c_int, ctypes.POINTER(_dp), ctypes.c_int,
                                ctypes.c_int, _dp]
        L.r1o_build_j.argtypes = [_dp, _u64p, ctypes.c_int, _dp, _dp]
        L.r1o_ldlt_factor.restype = ctypes.c_int
        L.r1o_ldlt_factor.argtypes = [ctypes.c_int64, _dp, _ip]
        L.r1o_ldlt_solve.argtypes = [ctypes.c_int64, _dp, _ip, _dp]
        L.r1o_ldlt_diag_condition.restype = ctypes.c_double
        L.r1o_ldlt_diag_condition.argtypes = [ctypes.c_int64, _dp, _ip, ctypes.c_int]
        L.r1o_rqi_step.restype = ctypes.c_int
        L.r1o_rqi_step.argtypes = [ctypes.c_int64, _dp, _dp, _dp]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(_dp)


def _dims(dims) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(dims, dtype=np.uint64))


# ---------------------------------------------------------------- inputs --

def rng_units(seed: int, stream: int, count: int, first: int = 0) -> np.ndarray:
    """CounterRng(seed, stream).next_unit() draws first+1..first+count (rng.hpp:17-20)."""
    out = np.empty(count)
    lib().r1o_rng_units(seed, stream, first, count, _p(out))
    return out


def rng_u64(seed: int, stream: int, count: int, first: int = 0) -> np.ndarray:
    out = np.empty(count, dtype=np.uint64)
    lib().r1o_rng_u64(seed, stream, first, count, out.ctypes.data_as(_u64p))
    return out


def rng_gaussians(seed: int, stream: int, count: int, first: int = 0) -> np.ndarray:
    """next_gaussian() values first..first+count-1 (generators.cpp:11-24)."""
    out = np.empty(count)
    lib().r1o_rng_gauss(seed, stream, first, count, _p(out))
    return out


def gen_gaussian(dims, seed: int) -> np.ndarray:
    """gen_gaussian (generators.cpp:50-56): stream kStreamTensor=1, layout order."""
    n = int(np.prod(dims))
    out = np.empty(n)
    lib().r1o_gen_gaussian(n, seed, _p(out))
    return out


def gen_config(cfg: int, dims, seed: int) -> np.ndarray:
    """BASELINE.json config tensor `cfg` (1..5) in reference dims; see rank1_oracle.c."""
    n = int(np.prod(dims))
    out = np.empty(n)
    d = _dims(dims)
    rc = lib().r1o_gen_config(cfg, d.ctypes.data_as(_u64p), len(dims), seed, _p(out))
    if rc != 0:
        raise ValueError(f"gen_config: unsupported config {cfg} for dims {tuple(dims)}")
    return out


def planted_factor(seed: int, k: int, length: int) -> np.ndarray:
    out = np.empty(length)
    lib().r1o_planted_factor(seed, k, length, _p(out))
    return out


def random_unit_factors(dims, seed: int, stream: int = 2) -> list[np.ndarray]:
    """solvers.cpp:34-49: uniform01 draws mode by mode from CounterRng(seed, stream),
    normalized (an all-zero draw becomes normalized ones)."""
    out, used = [], 0
    for n in dims:
        u = rng_units(seed, stream, n, first=used)
        used += n
        nrm = _norm2(u)
        if nrm == 0.0:
            u = np.ones(n)
            nrm = _norm2(u)
        out.append(u / nrm)
    return out


def oracle_random_tensor(dims, seed: int) -> np.ndarray:
    """tests/oracles.hpp:114-120 (stream 77)."""
    return rng_gaussians(seed, 77, int(np.prod(dims)))


def oracle_random_unit(n: int, seed: int) -> np.ndarray:
    """tests/oracles.hpp:122-128 (stream 78)."""
    v = rng_gaussians(seed, 78, n)
    return v / _norm2(v)


def oracle_random_unit_factors(dims, seed: int) -> list[np.ndarray]:
    """tests/oracles.hpp:130-137."""
    return [oracle_random_unit(n, seed * 131 + k) for k, n in enumerate(dims)]


def _norm2(v: np.ndarray) -> float:
    """matrix.cpp:62-66: sequential sum of squares."""
    s = 0.0
    for x in np.asarray(v, dtype=np.float64).tolist():
        s += x * x
    return math.sqrt(s)


# ------------------------------------------------------------- the sweep --

def pairs(d: int):
    return [(m, n) for m in range(d) for n in range(m + 1, d)]


def block_offsets(dims):
    offs, o = {}, 0
    for m, n in pairs(len(dims)):
        offs[(m, n)] = o
        o += dims[m] * dims[n]
    return offs, o


def build_j(a: np.ndarray, dims, factors) -> np.ndarray:
    """All P upper blocks with the reference's TTV-chain arithmetic
    (nepv.cpp:46-77, 199-231; tensor.cpp:100-138).  Bit-identical to the
    compiled reference (pinned in tests/test_oracle_pins.py)."""
    d = len(dims)
    _, total = block_offsets(dims)
    flat = np.ascontiguousarray(np.concatenate([np.asarray(f, dtype=np.float64) for f in factors]))
    out = np.empty(total)
    dd = _dims(dims)
    lib().r1o_build_j(_p(np.ascontiguousarray(a)), dd.ctypes.data_as(_u64p), d, _p(flat), _p(out))
    return out


def build_j_numpy(a: np.ndarray, dims, factors) -> np.ndarray:
    """Independent restatement by tensordot (different summation order) —
    a second witness for the block definition B(m,n) = A x_{k not in {m,n}} u_k."""
    d = len(dims)
    t = np.asarray(a).reshape(tuple(dims), order="F")
    blocks = []
    for m, n in pairs(d):
        r = t
        for k in reversed(range(d)):
            if k in (m, n):
                continue
            r = np.tensordot(r, factors[k], axes=([k], [0]))
        blocks.append(np.asarray(r).reshape(-1, order="F"))
    return np.concatenate(blocks) if blocks else np.empty(0)


def get_block(blocks: np.ndarray, dims, m: int, n: int) -> np.ndarray:
    offs, _ = block_offsets(dims)
    o = offs[(m, n)]
    return blocks[o:o + dims[m] * dims[n]].reshape(dims[m], dims[n], order="F")


def matvec(dims, blocks, x) -> np.ndarray:
    """SymBlockMatrix::matvec (nepv.cpp:110-134), scale 1/(d-1) included."""
    d = len(dims)
    off = np.concatenate([[0], np.cumsum(dims)]).astype(int)
    y = np.zeros(off[-1])
    x = np.asarray(x, dtype=np.float64)
    for m, n in pairs(d):
        b = get_block(blocks, dims, m, n)
        y[off[m]:off[m + 1]] += b @ x[off[n]:off[n + 1]]
        y[off[n]:off[n + 1]] += b.T @ x[off[m]:off[m + 1]]
    return y / (d - 1)


def dense(dims, blocks) -> np.ndarray:
    """SymBlockMatrix::dense (nepv.cpp:136-150)."""
    d = len(dims)
    off = np.concatenate([[0], np.cumsum(dims)]).astype(int)
    s = np.zeros((off[-1], off[-1]))
    sc = 1.0 / (d - 1)
    for m, n in pairs(d):
        b = get_block(blocks, dims, m, n) * sc
        s[off[m]:off[m + 1], off[n]:off[n + 1]] = b
        s[off[n]:off[n + 1], off[m]:off[m + 1]] = b.T
    return s


def frobenius(dims, blocks) -> float:
    """||J||_F = sqrt(2 sum ||B||^2) / (d-1) (nepv.cpp:152-157)."""
    return math.sqrt(2.0 * float(np.dot(blocks, blocks))) / (len(dims) - 1)


def scf_stopping_value(dims, blocks, x, lam: float) -> float:
    """Eq. 11 (nepv.cpp:271-282)."""
    y = matvec(dims, blocks, x)
    rho = float(np.dot(x, y))
    return float(np.linalg.norm(y - rho * np.asarray(x))) / (frobenius(dims, blocks) + abs(lam))


def kkt_from_blocks(dims, blocks, factors):
    """kkt_report (nepv.cpp:249-269) via the block identities: w_n = B(n,m) u_m
    (m != n), lambda = u_0' B(0,1) u_1.  Returns (lambda, max_res, per_mode)."""
    d = len(dims)
    if d == 2:
        b = get_block(blocks, dims, 0, 1)
        w = [b @ factors[1], b.T @ factors[0]]
    else:
        w = []
        for n in range(d):
            m = 1 if n == 0 else 0
            if m < n:
                w.append(get_block(blocks, dims, m, n).T @ factors[m])
            else:
                w.append(get_block(blocks, dims, n, m) @ factors[m])
    lam = float(np.dot(w[0], factors[0]))
    res = [float(np.linalg.norm(w[n] - lam * factors[n])) for n in range(d)]
    return lam, max(res), res


def multilinear_value(a, dims, factors) -> float:
    t = np.asarray(a).reshape(tuple(dims), order="F")
    r = t
    for k in reversed(range(len(dims))):
        r = np.tensordot(r, factors[k], axes=([k], [0]))
    return float(r)


# ------------------------------------------------------------ eigen steps --

def largest_magnitude_eigenpair(s: np.ndarray):
    """sym_eig.cpp:206-229 pick and sign rules on a LAPACK eigendecomposition."""
    w, v = np.linalg.eigh(s)
    lo, hi = 0, len(w) - 1
    pick = lo if abs(w[lo]) > abs(w[hi]) * (1.0 + 1e-12) else hi
    vec = v[:, pick].copy()
    arg = int(np.argmax(np.abs(vec)))  # first index wins ties, as :224-225
    if vec[arg] < 0.0:
        vec = -vec
    return float(w[pick]), vec


def rqi_step(s: np.ndarray, x: np.ndarray):
    """rayleigh_quotient_step (sym_eig.cpp:411-438) via the C restatement of
    Bunch-Kaufman; returns None for std::nullopt."""
    n = s.shape[0]
    sf = np.ascontiguousarray(np.asarray(s, dtype=np.float64).reshape(-1, order="F"))
    xx = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    y = np.empty(n)
    ok = lib().r1o_rqi_step(n, _p(sf), _p(xx), _p(y))
    return y if ok else None


def ldlt(s: np.ndarray):
    """(w, ipiv, singular, cond) of ldlt_factor / ldlt_diag_condition."""
    n = s.shape[0]
    w = np.ascontiguousarray(np.asarray(s, dtype=np.float64).reshape(-1, order="F")).copy()
    ipiv = np.zeros(n, dtype=np.int32)
    sing = lib().r1o_ldlt_factor(n, _p(w), ipiv.ctypes.data_as(_ip))
    cond = lib().r1o_ldlt_diag_condition(n, _p(w), ipiv.ctypes.data_as(_ip), sing)
    return w, ipiv, bool(sing), cond


# ---------------------------------------------------------- stacked ops --

def split_factors(dims, x):
    """split_factors (stacked.cpp:40-58): per-block normalize; <1e-12 -> zero + flag."""
    out, deg, o = [], [], 0
    for n in dims:
        blk = np.array(x[o:o + n], dtype=np.float64)
        o += n
        nrm = _norm2(blk)
        if nrm < 1e-12:
            out.append(np.zeros(n))
            deg.append(True)
        else:
            out.append(blk / nrm)
            deg.append(False)
    return out, deg


def stack_factors(factors) -> np.ndarray:
    """stack_factors (stacked.cpp:60-73): u/sqrt(d); throws if not unit to 1e-8."""
    d = len(factors)
    for u in factors:
        if abs(_norm2(u) - 1.0) > 1e-8:
            raise ValueError("stack_factors: factors must have unit norm")
    s = 1.0 / math.sqrt(d)
    return np.concatenate([np.asarray(u) * s for u in factors])


# ---------------------------------------------------------------- solvers --

@dataclass
class Options:
    tol: float = 1e-4
    max_iters: int = 500
    seed: int = 0
    init: str = "uniform01"
    init_factors: list | None = None
    rqi_accept_rule: str = "magnitude"
    record_kkt: bool = True
    scf_lambda_rtol: float = 0.0
    stop_rule: str = "kkt"           # baselines only (solvers.hpp:16, 25)
    asvd_disjoint_pairs: bool = False


@dataclass
class Report:
    algorithm: str
    lam: float = 0.0
    factors: list = field(default_factory=list)
    converged: bool = False
    iterations: int = 0
    lambda0: float = 0.0
    restarted: bool = False
    trace: list = field(default_factory=list)
    final_x: np.ndarray | None = None
    sweeps: int = 0


class _Degenerate(Exception):
    pass


def _initial(dims, opts: Options):
    if opts.init == "provided":
        f = []
        for n, u in zip(dims, opts.init_factors):
            u = np.asarray(u, dtype=np.float64)
            nrm = _norm2(u)
            if nrm == 0.0:
                raise ValueError("solver: provided init factor is zero")
            f.append(u / nrm)
        return f
    return random_unit_factors(dims, opts.seed, 2)


def _finalize(dims, blocks, u):
    lam, _, _ = kkt_from_blocks(dims, blocks, u)
    if lam < 0:
        lam = -lam
        u = [-u[0]] + list(u[1:])
    return lam, u


def _run(a, dims, opts: Options, u, accelerated: bool) -> Report:
    """run_hoscf (solvers.cpp:129-183) / run_ihoscf (:185-297) with the sweep
    J(u) from build_j; lambda0 / final lambda from the block identities."""
    rep = Report("ihoscf" if accelerated else "hoscf")
    j = build_j(a, dims, u)
    rep.sweeps = 1
    rep.lambda0 = kkt_from_blocks(dims, j, u)[0]
    lam_prev = None
    for k in range(1, opts.max_iters + 1):
        mu, vec = largest_magnitude_eigenpair(dense(dims, j))
        u_mid, deg = split_factors(dims, vec)
        if any(deg):
            raise _Degenerate()
        x_hat = stack_factors(u_mid)
        j_mid = build_j(a, dims, u_mid)
        rep.sweeps += 1
        rec = {"lambda": mu, "rqi_accepted": False, "lambda_pre_rqi": float("nan")}
        if not accelerated:
            u, j = u_mid, j_mid
            rec["eq11"] = scf_stopping_value(dims, j, x_hat, mu)
            rep.final_x = vec
        else:
            sv = scf_stopping_value(dims, j_mid, x_hat, mu)
            if sv <= opts.tol:
                rec["eq11"] = sv
                u, j = u_mid, j_mid
                rep.final_x = vec
            else:
                lam_mid = float(np.dot(x_hat, matvec(dims, j_mid, x_hat)))
                rec["lambda_pre_rqi"] = lam_mid
                accepted = False
                y = rqi_step(dense(dims, j_mid), x_hat)
                if y is not None:
                    u_r, deg_r = split_factors(dims, y)
                    if not any(deg_r):
                        rho_y = float(np.dot(y, matvec(dims, j_mid, y)))
                        better = (abs(rho_y) > abs(lam_mid)) if opts.rqi_accept_rule == "magnitude" \
                            else (rho_y > lam_mid)
                        if better:
                            accepted = True
                if accepted:
                    u = u_r
                    j = build_j(a, dims, u)
                    rep.sweeps += 1
                    rec["lambda"] = rho_y
                    rec["eq11"] = scf_stopping_value(dims, j, stack_factors(u), rho_y)
                    rep.final_x = y
                else:
                    u, j = u_mid, j_mid
                    rec["lambda"] = lam_mid
                    rec["eq11"] = sv
                    rep.final_x = vec
                rec["rqi_accepted"] = accepted
        rec["stop_value"] = rec["eq11"]
        rec["kkt"] = kkt_from_blocks(dims, j, u)[1] if opts.record_kkt else float("nan")
        rep.trace.append(rec)
        rep.iterations = k
        if rec["stop_value"] <= opts.tol:
            rep.converged = True
            break
        if opts.scf_lambda_rtol > 0 and lam_prev is not None and \
                abs(rec["lambda"] - lam_prev) <= opts.scf_lambda_rtol * abs(rec["lambda"]):
            break
        lam_prev = rec["lambda"]
    rep.lam, rep.factors = _finalize(dims, j, u)
    return rep


# ------------------------------------------------------------- baselines --

def contract_leaving(a, dims, factors, mode: int) -> np.ndarray:
    """contract_leaving (tensor.cpp:220-233): A contracted with every factor but
    `mode` (tensordot chain, highest mode first like ttvc, :157-170)."""
    r = np.asarray(a).reshape(tuple(dims), order="F")
    for k in reversed(range(len(dims))):
        if k != mode:
            r = np.tensordot(r, factors[k], axes=([k], [0]))
    return np.asarray(r, dtype=np.float64).reshape(-1)


def build_block(a, dims, factors, m: int, n: int) -> np.ndarray:
    """build_block (nepv.hpp:54): I_m x I_n matrix A x_{k not in {m,n}} u_k."""
    r = np.asarray(a).reshape(tuple(dims), order="F")
    for k in reversed(range(len(dims))):
        if k not in (m, n):
            r = np.tensordot(r, factors[k], axes=([k], [0]))
    return np.asarray(r, dtype=np.float64)


def top_singular_pair(b: np.ndarray):
    """top_singular_pair (solvers.cpp:358-381) via the [[0,B],[B',0]] embedding."""
    r, c = b.shape
    e = np.zeros((r + c, r + c))
    e[:r, r:] = b
    e[r:, :r] = b.T
    val, vec = largest_magnitude_eigenpair(e)
    if val < 0.0:
        vec = vec.copy()
        vec[r:] = -vec[r:]
        val = -val
    left, right = vec[:r].copy(), vec[r:].copy()
    nl, nr = _norm2(left), _norm2(right)
    if nl > 0:
        left /= nl
    if nr > 0:
        right /= nr
    if nl < 1e-12 or nr < 1e-12:
        raise _Degenerate()
    return val, left, right


def asvd_pairs(d: int, disjoint: bool, iteration: int):
    """asvd_pairs (solvers.cpp:383-397)."""
    if disjoint:
        off = (iteration - 1) % 2 if d > 2 else 0
        return [(m, m + 1) for m in range(off, d - 1, 2)]
    pairs = [(m, m + 1) for m in range(d - 1)]
    if d > 2:
        pairs.append((0, d - 1))
    return pairs


def _baseline_stop(a, dims, u, lam, lam_prev, a_norm, opts: Options):
    """baseline_stop (solvers.cpp:100-127): (value, eq11, kkt_max)."""
    blocks = build_j(a, dims, u) if len(dims) > 2 else np.asarray(a, dtype=np.float64).copy()
    _, kkt_max, _ = kkt_from_blocks(dims, blocks, u)
    nan = float("nan")
    if opts.stop_rule == "eq11":
        eq = scf_stopping_value(dims, blocks, stack_factors(u), lam)
        return eq, eq, (kkt_max if opts.record_kkt else nan)
    if opts.stop_rule == "lambda_delta":
        v = abs(lam - lam_prev) / max(abs(lam), 1e-300)
        return v, nan, (kkt_max if opts.record_kkt else nan)
    return kkt_max / max(a_norm, 1e-300), nan, kkt_max


def _run_baseline(a, dims, opts: Options, u, kind: str) -> Report:
    """run_power_sweep (solvers.cpp:299-354) / run_asvd (:400-447)."""
    rep = Report(kind)
    d = len(dims)
    u = [np.asarray(x, dtype=np.float64).copy() for x in u]
    rep.lambda0 = multilinear_value(a, dims, u)
    a_norm = float(np.sqrt(np.dot(a, a)))
    lam_prev = rep.lambda0
    for k in range(1, opts.max_iters + 1):
        if kind == "hopm":
            for n in range(d):
                w = contract_leaving(a, dims, u, n)
                nrm = _norm2(w)
                if nrm < 1e-300:
                    raise _Degenerate()
                u[n] = w / nrm
                lam = nrm
        elif kind == "jacobi_hopm":
            ws = [contract_leaving(a, dims, u, n) for n in range(d)]
            for n in range(d):
                nrm = _norm2(ws[n])
                if nrm < 1e-300:
                    raise _Degenerate()
                u[n] = ws[n] / nrm
            lam = multilinear_value(a, dims, u)
        else:
            jacobi = kind == "jacobi_asvd"
            snap = [x.copy() for x in u]
            nxt = [x.copy() for x in u]
            for m, n in asvd_pairs(d, opts.asvd_disjoint_pairs, k):
                src = snap if jacobi else nxt
                _, left, right = top_singular_pair(build_block(a, dims, src, m, n))
                nxt[m], nxt[n] = left, right
            u = nxt
            lam = multilinear_value(a, dims, u)
        value, eq, kkt = _baseline_stop(a, dims, u, lam, lam_prev, a_norm, opts)
        rep.trace.append({"lambda": lam, "stop_value": value, "eq11": eq, "kkt": kkt})
        rep.iterations = k
        lam_prev = lam
        if value <= opts.tol:
            rep.converged = True
            break
    lam = multilinear_value(a, dims, u)
    if lam < 0:
        lam = -lam
        u[0] = -u[0]
    rep.lam, rep.factors = lam, u
    return rep


def _solve(a, dims, opts: Options, accelerated) -> Report:
    """validate + with_restart (solvers.cpp:28-32, 78-91)."""
    if len(dims) < 2:
        raise ValueError("solver: tensor order must be >= 2")
    if not opts.tol > 0.0:
        raise ValueError("solver: tol must be > 0")
    if opts.max_iters < 1:
        raise ValueError("solver: max_iters must be >= 1")
    def go(u):
        if isinstance(accelerated, str):
            return _run_baseline(a, dims, opts, u, accelerated)
        return _run(a, dims, opts, u, accelerated)

    try:
        return go(_initial(dims, opts))
    except _Degenerate:
        try:
            rep = go(random_unit_factors(dims, opts.seed, 3))
            rep.restarted = True
            return rep
        except _Degenerate as e:
            raise RuntimeError("solver failed after restart") from e


def hoscf(a, dims, opts: Options) -> Report:
    return _solve(a, dims, opts, False)


def ihoscf(a, dims, opts: Options) -> Report:
    return _solve(a, dims, opts, True)


def hopm(a, dims, opts: Options) -> Report:
    return _solve(a, dims, opts, "hopm")


def jacobi_hopm(a, dims, opts: Options) -> Report:
    return _solve(a, dims, opts, "jacobi_hopm")


def asvd(a, dims, opts: Options) -> Report:
    return _solve(a, dims, opts, "asvd")


def jacobi_asvd(a, dims, opts: Options) -> Report:
    return _solve(a, dims, opts, "jacobi_asvd")


# ------------------------------------------------------- greedy deflation --

def rank_one_expand(lam, factors, dims) -> np.ndarray:
    """rank_one_expand (tensor.cpp:246-265): buf = [lambda]; mode by mode
    next[i |buf| + p] = buf[p] u_n[i] — the left-to-right product."""
    buf = np.array([lam], dtype=np.float64)
    for n, d in enumerate(dims):
        u = np.asarray(factors[n], dtype=np.float64)
        buf = np.outer(u, buf).reshape(-1)  # next[i * |buf| + p] = u[i] * buf[p]
    return buf


def greedy_rank_r(a, dims, r, solver: str, opts: Options):
    """greedy_rank_r (greedy.cpp:7-35): returns dict(lambdas, terms, ratios,
    iterations, completed, failure)."""
    if r < 1:
        raise ValueError("greedy_rank_r: rank must be >= 1")
    a = np.asarray(a, dtype=np.float64)
    base = float(np.sqrt(np.dot(a, a)))
    if base == 0.0:
        raise ValueError("greedy_rank_r: zero input tensor")
    res = a.copy()
    out = dict(lambdas=[], terms=[], ratios=[], iterations=[], completed=False, failure="")
    fn = {"hoscf": hoscf, "ihoscf": ihoscf, "hopm": hopm, "jacobi_hopm": jacobi_hopm,
          "asvd": asvd, "jacobi_asvd": jacobi_asvd}[solver]
    for term in range(r):
        o = Options(**{**opts.__dict__, "seed": opts.seed + term})
        try:
            rep = fn(res, dims, o)
        except Exception as e:  # greedy.cpp:19-23
            out["failure"] = f"term {term + 1}: {e}"
            return out
        res = res - rank_one_expand(rep.lam, rep.factors, dims)
        out["lambdas"].append(rep.lam)
        out["terms"].append([np.asarray(u).copy() for u in rep.factors])
        out["ratios"].append(float(np.sqrt(np.dot(res, res))) / base)
        out["iterations"].append(rep.iterations)
    out["completed"] = True
    return out


# ------------------------------------------------------------------ .dt1 --

DT1_MAGIC = b"DTEN1\0"


def write_dt1(path, a, dims) -> None:
    """write_dt1 (tensor_io.cpp:47-64): magic, u8 order, u64le dims, f64le payload."""
    if len(dims) < 2:
        raise ValueError("write_dt1: tensor order must be >= 2")
    with open(path, "wb") as f:
        f.write(DT1_MAGIC)
        f.write(bytes([len(dims)]))
        for d in dims:
            f.write(int(d).to_bytes(8, "little"))
        f.write(np.ascontiguousarray(a, dtype="<f8").tobytes())


def read_dt1(path):
    """read_dt1 (tensor_io.cpp:66-100) with the same checks and messages."""
    try:
        f = open(path, "rb")
    except OSError:
        raise RuntimeError(f"read_dt1: cannot open {path}")
    with f:
        if f.read(6) != DT1_MAGIC:
            raise RuntimeError(f"read_dt1: bad magic in {path}")
        b = f.read(1)
        if len(b) != 1 or b[0] < 2:
            raise RuntimeError("read_dt1: tensor order must be >= 2")
        dims, count = [], 1
        for _ in range(b[0]):
            v = f.read(8)
            d = int.from_bytes(v, "little") if len(v) == 8 else 0
            if d == 0:
                raise RuntimeError("read_dt1: invalid dimension")
            if count > (2 ** 64 - 1) // d:
                raise RuntimeError("read_dt1: size overflow")
            dims.append(d)
            count *= d
        payload = f.read()
    if len(payload) < 8 * count:
        raise RuntimeError(f"read_dt1: truncated payload in {path}")
    if len(payload) > 8 * count:
        raise RuntimeError(f"read_dt1: trailing bytes in {path}")
    return np.frombuffer(payload, dtype="<f8").astype(np.float64), dims
