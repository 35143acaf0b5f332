"""ORACLE / TEST INFRASTRUCTURE — ctypes binding of the compiled, unmodified
reference (oracle/_ref/librank1_ref.so, built by oracle/Makefile from
/root/reference/proj/src + oracle/ref_shim.cpp).

Used only by tests/ (parity checker), __graft_entry__.smoke() and bench.py's
CPU baseline / `--impl reference` arm.  `available()` is False on hosts where
the .so was never built (it is git-ignored; it travels to GPU boxes with the
gpurun snapshot).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "librank1_ref.so")
_lib = None

_dp = ctypes.POINTER(ctypes.c_double)
_u64p = ctypes.POINTER(ctypes.c_uint64)
_ip = ctypes.POINTER(ctypes.c_int)


class RefError(Exception):
    pass


class RefInvalidArgument(RefError, ValueError):
    pass


class RefRuntimeError(RefError, RuntimeError):
    pass


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise RefError(f"reference oracle not built: {LIB_PATH} (run make -C oracle)")
        _lib = ctypes.CDLL(LIB_PATH)
        _lib.ref_last_error.restype = ctypes.c_char_p
    return _lib


def _check(rc: int):
    if rc == 0:
        return
    msg = lib().ref_last_error().decode()
    if rc == 1:
        raise RefInvalidArgument(msg)
    if rc == 2:
        raise RefRuntimeError(msg)
    raise RefError(msg)


def _d(a):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    return a, a.ctypes.data_as(_dp)


def _dims(dims):
    d = np.ascontiguousarray(np.asarray(dims, dtype=np.uint64))
    return d, d.ctypes.data_as(_u64p)


def max_threads() -> int:
    return int(lib().ref_max_threads())


def blocks_numel(dims) -> int:
    d = len(dims)
    return sum(dims[m] * dims[n] for m in range(d) for n in range(m + 1, d))


def build_j(a, dims, factors, serial=False, threads=0, determinism=True, reuse=False):
    a, ap = _d(a)
    dd, dp = _dims(dims)
    flat, fp = _d(np.concatenate([np.asarray(f, dtype=np.float64) for f in factors]))
    out = np.empty(blocks_numel(dims))
    secs = ctypes.c_double()
    _check(lib().ref_build_j(ap, dp, len(dims), fp, 1 if serial else 0, threads,
                             1 if determinism else 0, 1 if reuse else 0,
                             out.ctypes.data_as(_dp), ctypes.byref(secs)))
    return out


def time_build_j(a, dims, factors, reps=3, threads=0, determinism=True):
    """(blocks, per-call seconds) with the tensor copied into the reference's
    DenseTensor once, outside the timed calls."""
    a, ap = _d(a)
    dd, dp = _dims(dims)
    flat, fp = _d(np.concatenate([np.asarray(f, dtype=np.float64) for f in factors]))
    out = np.empty(blocks_numel(dims))
    secs = np.zeros(reps)
    _check(lib().ref_time_build_j(ap, dp, len(dims), fp, threads, 1 if determinism else 0, reps,
                                  out.ctypes.data_as(_dp), secs.ctypes.data_as(_dp)))
    return out, secs


def build_block(a, dims, factors, m, n):
    a, ap = _d(a)
    dd, dp = _dims(dims)
    flat, fp = _d(np.concatenate([np.asarray(f, dtype=np.float64) for f in factors]))
    mm, nn = min(m, n), max(m, n)
    out = np.empty(dims[mm] * dims[nn])
    _check(lib().ref_build_block(ap, dp, len(dims), fp, m, n, out.ctypes.data_as(_dp)))
    return out


def multilinear_value(a, dims, factors) -> float:
    a, ap = _d(a)
    dd, dp = _dims(dims)
    flat, fp = _d(np.concatenate([np.asarray(f, dtype=np.float64) for f in factors]))
    v = ctypes.c_double()
    _check(lib().ref_multilinear_value(ap, dp, len(dims), fp, ctypes.byref(v)))
    return v.value


def kkt_report(a, dims, factors):
    a, ap = _d(a)
    dd, dp = _dims(dims)
    flat, fp = _d(np.concatenate([np.asarray(f, dtype=np.float64) for f in factors]))
    out = np.empty(len(dims) + 2)
    _check(lib().ref_kkt_report(ap, dp, len(dims), fp, out.ctypes.data_as(_dp)))
    return float(out[0]), float(out[1]), out[2:].tolist()


def block_matvec(dims, blocks, x):
    dd, dp = _dims(dims)
    b, bp = _d(blocks)
    xx, xp = _d(x)
    y = np.empty(sum(dims))
    _check(lib().ref_block_matvec(dp, len(dims), bp, xp, y.ctypes.data_as(_dp)))
    return y


def block_frobenius(dims, blocks) -> float:
    dd, dp = _dims(dims)
    b, bp = _d(blocks)
    v = ctypes.c_double()
    _check(lib().ref_block_frobenius(dp, len(dims), bp, ctypes.byref(v)))
    return v.value


def block_dense(dims, blocks):
    dd, dp = _dims(dims)
    b, bp = _d(blocks)
    n = sum(dims)
    out = np.empty(n * n)
    _check(lib().ref_block_dense(dp, len(dims), bp, out.ctypes.data_as(_dp)))
    return out.reshape(n, n, order="F")


def scf_stopping_value(dims, blocks, x, lam) -> float:
    dd, dp = _dims(dims)
    b, bp = _d(blocks)
    xx, xp = _d(x)
    v = ctypes.c_double()
    _check(lib().ref_scf_stopping_value(dp, len(dims), bp, xp, ctypes.c_double(lam),
                                        ctypes.byref(v)))
    return v.value


def _mat(s):
    s = np.asarray(s, dtype=np.float64)
    n = s.shape[0]
    f = np.ascontiguousarray(s.reshape(-1, order="F"))
    return n, f, f.ctypes.data_as(_dp)


def sym_eig_full(s):
    n, f, fp = _mat(s)
    w = np.empty(n)
    v = np.empty(n * n)
    _check(lib().ref_sym_eig_full(ctypes.c_int64(n), fp, w.ctypes.data_as(_dp),
                                  v.ctypes.data_as(_dp)))
    return w, v.reshape(n, n, order="F")


def largest_magnitude_eigenpair(s):
    n, f, fp = _mat(s)
    val = ctypes.c_double()
    vec = np.empty(n)
    _check(lib().ref_largest_magnitude_eigenpair(ctypes.c_int64(n), fp, ctypes.byref(val),
                                                 vec.ctypes.data_as(_dp)))
    return val.value, vec


def rayleigh_quotient_step(s, x):
    n, f, fp = _mat(s)
    xx, xp = _d(x)
    y = np.empty(n)
    acc = ctypes.c_int()
    _check(lib().ref_rayleigh_quotient_step(ctypes.c_int64(n), fp, xp, y.ctypes.data_as(_dp),
                                            ctypes.byref(acc)))
    return y if acc.value else None


def ldlt(s):
    n, f, fp = _mat(s)
    w = np.empty(n * n)
    ipiv = np.empty(n, dtype=np.int32)
    sing = ctypes.c_int()
    cond = ctypes.c_double()
    _check(lib().ref_ldlt(ctypes.c_int64(n), fp, w.ctypes.data_as(_dp),
                          ipiv.ctypes.data_as(_ip), ctypes.byref(sing), ctypes.byref(cond)))
    return w.reshape(n, n, order="F"), ipiv, bool(sing.value), cond.value


def split_factors(dims, x):
    dd, dp = _dims(dims)
    xx, xp = _d(x)
    f = np.empty(sum(dims))
    deg = np.zeros(len(dims), dtype=np.uint8)
    _check(lib().ref_split_factors(dp, len(dims), xp, f.ctypes.data_as(_dp),
                                   deg.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))))
    offs = np.concatenate([[0], np.cumsum(dims)]).astype(int)
    return [f[offs[k]:offs[k + 1]] for k in range(len(dims))], [bool(v) for v in deg]


def stack_factors(dims, factors):
    dd, dp = _dims(dims)
    flat, fp = _d(np.concatenate([np.asarray(f, dtype=np.float64) for f in factors]))
    x = np.empty(sum(dims))
    _check(lib().ref_stack_factors(dp, len(dims), fp, x.ctypes.data_as(_dp)))
    return x


def gen_gaussian(dims, seed):
    dd, dp = _dims(dims)
    out = np.empty(int(np.prod(dims)))
    _check(lib().ref_gen_gaussian(dp, len(dims), ctypes.c_uint64(seed), out.ctypes.data_as(_dp)))
    return out


def generate(name, dims, seed=0):
    dd, dp = _dims(dims)
    out = np.empty(int(np.prod(dims)))
    _check(lib().ref_generate(name.encode(), dp, len(dims), ctypes.c_uint64(seed),
                              out.ctypes.data_as(_dp)))
    return out


def rng_draws(seed, stream, kind, count):
    out = np.empty(count)
    _check(lib().ref_rng_draws(ctypes.c_uint64(seed), ctypes.c_uint64(stream), kind,
                               ctypes.c_int64(count), out.ctypes.data_as(_dp)))
    if kind == 0:
        return out.view(np.uint64)
    return out


# --- solve(): uses the product header's POD structs, mirrored here --------

class SolveOptionsC(ctypes.Structure):
    _fields_ = [("tol", ctypes.c_double), ("max_iters", ctypes.c_int32),
                ("init", ctypes.c_int32), ("seed", ctypes.c_uint64),
                ("init_factors", _dp), ("determinism", ctypes.c_int32),
                ("rqi_accept_rule", ctypes.c_int32), ("stop_rule", ctypes.c_int32),
                ("threads", ctypes.c_int32), ("record_kkt", ctypes.c_int32),
                ("asvd_disjoint_pairs", ctypes.c_int32),
                ("reuse_intermediates", ctypes.c_int32), ("scf_lambda_rtol", ctypes.c_double),
                ("scf_angle_tol", ctypes.c_double)]


class IterationRecordC(ctypes.Structure):
    _fields_ = [("lambda_", ctypes.c_double), ("stop_value", ctypes.c_double),
                ("eq11_value", ctypes.c_double), ("kkt_max_residual", ctypes.c_double),
                ("rqi_accepted", ctypes.c_int32), ("n_sweeps", ctypes.c_int32),
                ("lambda_pre_rqi", ctypes.c_double), ("t_build_j", ctypes.c_double),
                ("t_eig", ctypes.c_double), ("t_other", ctypes.c_double),
                ("factor_change", ctypes.c_double)]


class SolveReportC(ctypes.Structure):
    _fields_ = [("lambda_", ctypes.c_double), ("factors", _dp), ("converged", ctypes.c_int32),
                ("iterations", ctypes.c_int32), ("lambda0", ctypes.c_double),
                ("restarted", ctypes.c_int32), ("final_x", _dp),
                ("trace", ctypes.POINTER(IterationRecordC)), ("total_sweeps", ctypes.c_int32),
                ("t_total", ctypes.c_double)]


def _solve_opts(tol, max_iters, seed, init_factors, rqi_accept_rule, record_kkt, determinism,
                threads, stop_rule, asvd_disjoint_pairs):
    o = SolveOptionsC()
    o.tol = tol
    o.max_iters = max_iters
    o.seed = seed
    o.determinism = 1 if determinism else 0
    o.rqi_accept_rule = rqi_accept_rule
    o.record_kkt = 1 if record_kkt else 0
    o.threads = threads
    o.stop_rule = stop_rule
    o.asvd_disjoint_pairs = 1 if asvd_disjoint_pairs else 0
    keep = None
    if init_factors is not None:
        keep = np.ascontiguousarray(np.concatenate([np.asarray(f, dtype=np.float64)
                                                    for f in init_factors]))
        o.init = 1
        o.init_factors = keep.ctypes.data_as(_dp)
    return o, keep


def _solve_call(call, dims, max_iters):
    n = sum(dims)
    fac = np.empty(n)
    fx = np.empty(n)
    tr = (IterationRecordC * max_iters)()
    r = SolveReportC()
    r.factors = fac.ctypes.data_as(_dp)
    r.final_x = fx.ctypes.data_as(_dp)
    r.trace = tr
    _check(call(ctypes.byref(r)))
    offs = np.concatenate([[0], np.cumsum(dims)]).astype(int)
    trace = []
    for i in range(r.iterations):
        t = tr[i]
        trace.append(dict(lambda_=t.lambda_, stop_value=t.stop_value, eq11=t.eq11_value,
                          kkt=t.kkt_max_residual, rqi_accepted=bool(t.rqi_accepted),
                          lambda_pre_rqi=t.lambda_pre_rqi, t_build_j=t.t_build_j,
                          t_eig=t.t_eig, t_other=t.t_other))
    return dict(lam=r.lambda_, factors=[fac[offs[k]:offs[k + 1]].copy() for k in range(len(dims))],
                converged=bool(r.converged), iterations=r.iterations, lambda0=r.lambda0,
                restarted=bool(r.restarted), final_x=fx.copy(), trace=trace,
                sweeps=r.total_sweeps, seconds=r.t_total)


def solve(algorithm, a, dims, tol=1e-4, max_iters=500, seed=0, init_factors=None,
          rqi_accept_rule=0, record_kkt=True, determinism=True, threads=0, stop_rule=0,
          asvd_disjoint_pairs=False):
    """rank1::solve through the reference; returns a dict mirroring SolveReport."""
    a, ap = _d(a)
    dd, dp = _dims(dims)
    o, keep = _solve_opts(tol, max_iters, seed, init_factors, rqi_accept_rule, record_kkt,
                          determinism, threads, stop_rule, asvd_disjoint_pairs)
    return _solve_call(lambda rp: lib().ref_solve(algorithm.encode(), ap, dp, len(dims),
                                                  ctypes.byref(o), rp), dims, max_iters)


_FILL = ctypes.CFUNCTYPE(None, _dp, ctypes.c_uint64, ctypes.c_void_p)


def solve_fill(algorithm, fill, dims, tol=1e-4, max_iters=500, seed=0, init_factors=None,
               rqi_accept_rule=0, record_kkt=True, determinism=True, threads=0, stop_rule=0):
    """rank1::solve on a tensor the reference allocates itself (DenseTensor(dims))
    and `fill(address, numel)` writes in place — one host copy of the tensor."""
    dd, dp = _dims(dims)
    o, keep = _solve_opts(tol, max_iters, seed, init_factors, rqi_accept_rule, record_kkt,
                          determinism, threads, stop_rule, False)
    cb = _FILL(lambda ptr, n, user: fill(ctypes.cast(ptr, ctypes.c_void_p).value, int(n)))
    return _solve_call(lambda rp: lib().ref_solve_fill(algorithm.encode(), cb, None, dp, len(dims),
                                                       ctypes.byref(o), rp), dims, max_iters)


def greedy(solver, a, dims, r, tol=1e-4, max_iters=500, seed=0, stop_rule=0):
    """rank1::greedy_rank_r through the reference."""
    a, ap = _d(a)
    dd, dp = _dims(dims)
    o = SolveOptionsC()
    o.tol, o.max_iters, o.seed, o.determinism, o.record_kkt = tol, max_iters, seed, 1, 1
    o.stop_rule = stop_rule
    n = sum(dims)
    lam = np.zeros(r)
    fac = np.zeros(r * n)
    rat = np.zeros(r)
    its = np.zeros(r, dtype=np.int32)
    nt, comp = ctypes.c_int(), ctypes.c_int()
    fail = ctypes.create_string_buffer(512)
    _check(lib().ref_greedy(solver.encode(), ap, dp, len(dims), ctypes.c_uint64(r), ctypes.byref(o),
                            lam.ctypes.data_as(_dp), fac.ctypes.data_as(_dp),
                            rat.ctypes.data_as(_dp), its.ctypes.data_as(_ip), ctypes.byref(nt),
                            ctypes.byref(comp), fail, 512))
    k = nt.value
    offs = np.concatenate([[0], np.cumsum(dims)]).astype(int)
    terms = [[fac[i * n + offs[m]:i * n + offs[m + 1]].copy() for m in range(len(dims))]
             for i in range(k)]
    return dict(lambdas=lam[:k].copy(), terms=terms, ratios=rat[:k].copy(),
                iterations=its[:k].tolist(), completed=bool(comp.value),
                failure=fail.value.decode())


def write_dt1(path, a, dims):
    a, ap = _d(a)
    dd, dp = _dims(dims)
    _check(lib().ref_write_dt1(str(path).encode(), ap, dp, len(dims)))


def read_dt1(path):
    dims = (ctypes.c_uint64 * 256)()
    order = ctypes.c_int()
    _check(lib().ref_read_dt1(str(path).encode(), dims, ctypes.byref(order), None, ctypes.c_uint64(0)))
    d = [int(dims[k]) for k in range(order.value)]
    out = np.empty(int(np.prod(d)))
    _check(lib().ref_read_dt1(str(path).encode(), dims, ctypes.byref(order), out.ctypes.data_as(_dp),
                              ctypes.c_uint64(out.size)))
    return out, d


def experiment_csv(generator, a, dims, algos, seeds, base_seed=0, tol=1e-4, max_iters=500):
    """run_experiment + experiment_csv(zero_timings) + summary_table of the reference."""
    a, ap = _d(a)
    dd, dp = _dims(dims)
    o = SolveOptionsC()
    o.tol, o.max_iters, o.determinism, o.record_kkt = tol, max_iters, 1, 1
    buf = ctypes.create_string_buffer(1 << 20)
    _check(lib().ref_experiment_csv(generator.encode(), ap, dp, len(dims), ",".join(algos).encode(),
                                    ctypes.c_uint64(seeds), ctypes.c_uint64(base_seed),
                                    ctypes.byref(o), buf, 1 << 20))
    csv_text, _, table = buf.value.decode().partition("\n\n")
    return csv_text + "\n", table


class RefTensor:
    """A reference DenseTensor allocated by the reference library and filled in
    place by `fill(address, numel)` (oracle/ref_shim.cpp ref_tensor_new): one host
    copy, generated once, reused by several timed calls (bench.py CPU arms)."""

    def __init__(self, fill, dims):
        self.dims = tuple(int(v) for v in dims)
        self._dd, dp = _dims(self.dims)
        L = lib()
        L.ref_tensor_data.restype = ctypes.c_void_p
        self._cb = _FILL(lambda ptr, n, user: fill(ctypes.cast(ptr, ctypes.c_void_p).value, int(n)))
        h = ctypes.c_void_p()
        _check(L.ref_tensor_new(self._cb, None, dp, len(self.dims), ctypes.byref(h)))
        self.handle = h

    def close(self):
        if self.handle:
            lib().ref_tensor_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def time_build_j(self, factors, reps=1, threads=0, determinism=True, want_blocks=False):
        """Per-call wall seconds of rank1::build_j (and the last call's blocks)."""
        flat, fp = _d(np.concatenate([np.asarray(f, dtype=np.float64) for f in factors]))
        out = np.empty(blocks_numel(self.dims)) if want_blocks else None
        secs = np.zeros(reps)
        _check(lib().ref_time_build_j_t(self.handle, fp, threads, 1 if determinism else 0, reps,
                                        out.ctypes.data_as(_dp) if out is not None else None,
                                        secs.ctypes.data_as(_dp)))
        return out, secs

    def solve(self, algorithm, tol=1e-4, max_iters=500, seed=0, init_factors=None,
              rqi_accept_rule=0, record_kkt=True, determinism=True, threads=0, stop_rule=0):
        o, keep = _solve_opts(tol, max_iters, seed, init_factors, rqi_accept_rule, record_kkt,
                              determinism, threads, stop_rule, False)
        return _solve_call(lambda rp: lib().ref_solve_t(algorithm.encode(), self.handle,
                                                        ctypes.byref(o), rp), self.dims, max_iters)
