// Dense-matrix entry points of the drop-in that the solvers' hot path does not
// use but the reference's API exports (sym_eig.hpp:11-54, tensor.hpp:55-58):
//
//   sym_eig_full                 Householder tridiagonalisation with accumulated
//                                transforms + implicit-shift QL + ascending sort
//                                (sym_eig.cpp:27-186, 188-204)
//   largest_magnitude_eigenpair  its pick / sign rules on that decomposition
//                                (sym_eig.cpp:206-229)
//   detail::ldlt_factor / _solve / _diag_condition
//                                unblocked Bunch-Kaufman in the reference's
//                                storage convention (sym_eig.cpp:233-407)
//   matricize / dematricize      mode-n unfoldings (tensor.cpp:72-98)
//   ttv / ttvc / ttvc_scalar     single-mode contraction chains (tensor.cpp:100-199):
//                                one thread per output entry, each summing its
//                                fibre in the reference's ascending order
//
// All of them run on the device in ONE thread block: every elementwise update
// is spread over the block's threads, while each sum the reference forms
// sequentially is formed by one thread in the same order, and this file is
// compiled with -fmad=false (no FMA contraction: the reference is built
// without -march=native).  The results therefore follow the reference's
// rounding step for step (only std::hypot / sqrt may differ in the last ulp
// between glibc and libdevice).  One block bounds the bandwidth to ~100 GB/s
// (sym_eig_full n = 3000: ~2 s, the reference: ~50 s); the solvers never call
// these — their eigen step is the Lanczos of lanczos.cu and their RQI the
// blocked Bunch-Kaufman of bk.cu.
#include "common.cuh"

#include <algorithm>
#include <cmath>
#include <vector>

namespace r1 {

namespace {

constexpr int kDenseThreads = 1024;
constexpr int kMaxQlSweeps = 60;  // sym_eig.cpp:11

__device__ __forceinline__ double& at(double* V, int64_t n, int64_t r, int64_t c) {
    return V[r + c * n];
}

// status: 0 ok, 1 QL did not converge
struct SymEigArgs {
    double* V;   // n x n, in: S (lower triangle read), out: eigenvectors
    double* d;   // n: out eigenvalues (ascending)
    double* e;   // n scratch
    double* cs;  // n scratch: rotation cosines of one QL sweep
    double* sn;  // n scratch: rotation sines
    int64_t n;
    int* status;
};

__global__ void __launch_bounds__(kDenseThreads) sym_eig_kernel(SymEigArgs a) {
    const int64_t n = a.n;
    double* V = a.V;
    double* d = a.d;
    double* e = a.e;
    const int tid = threadIdx.x;
    const int T = blockDim.x;
    __shared__ double sh[4];
    __shared__ int64_t shm[2];
    __shared__ int flag[2];

    // The reference reads only the lower triangle of the active block; keep a
    // mirror in the upper triangle so that every thread walks its own row with
    // coalesced loads (column-major: row r, column c at r + c n).
    for (int64_t idx = tid; idx < n * n; idx += T) {
        const int64_t r = idx % n, c = idx / n;
        if (r < c) V[idx] = at(V, n, c, r);
    }
    __syncthreads();

    // ---- Householder reduction (tridiagonalize, sym_eig.cpp:27-83) ----------
    for (int64_t j = tid; j < n; j += T) d[j] = at(V, n, n - 1, j);
    __syncthreads();
    for (int64_t i = n - 1; i > 0; --i) {
        if (tid == 0) {
            double scale = 0.0;
            for (int64_t k = 0; k < i; ++k) scale += fabs(d[k]);
            sh[0] = scale;
        }
        __syncthreads();
        const double scale = sh[0];
        double h = 0.0;
        if (scale == 0.0) {
            if (tid == 0) e[i] = d[i - 1];
            __syncthreads();
            for (int64_t j = tid; j < i; j += T) {
                d[j] = at(V, n, i - 1, j);
                at(V, n, i, j) = 0.0;
                at(V, n, j, i) = 0.0;
            }
        } else {
            for (int64_t k = tid; k < i; k += T) d[k] /= scale;
            __syncthreads();
            if (tid == 0) {
                double hh = 0.0;
                for (int64_t k = 0; k < i; ++k) hh += d[k] * d[k];
                const double f = d[i - 1];
                double g = sqrt(hh);
                if (f > 0) g = -g;
                e[i] = scale * g;
                hh -= f * g;
                d[i - 1] = f - g;
                sh[1] = hh;
            }
            __syncthreads();
            h = sh[1];
            // e = A d over the active block (row r: the reference's sequence of
            // products A(r, j) d_j, j ascending), Householder vector into column i
            for (int64_t r = tid; r < i; r += T) {
                at(V, n, r, i) = d[r];
                double acc = 0.0;
                for (int64_t j = 0; j < i; ++j) acc += at(V, n, r, j) * d[j];
                e[r] = acc;
            }
            __syncthreads();
            for (int64_t j = tid; j < i; j += T) e[j] /= h;
            __syncthreads();
            if (tid == 0) {
                double f = 0.0;
                for (int64_t j = 0; j < i; ++j) f += e[j] * d[j];
                sh[2] = f / (h + h);
            }
            __syncthreads();
            const double hh = sh[2];
            for (int64_t j = tid; j < i; j += T) e[j] -= hh * d[j];
            __syncthreads();
            // rank-2 update v(k, j) -= d_j e_k + e_j d_k (k >= j) and its mirror
            for (int64_t r = tid; r < i; r += T) {
                const double dr = d[r], er = e[r];
                for (int64_t c = 0; c < i; ++c) {
                    const double s = c <= r ? d[c] * er + e[c] * dr : dr * e[c] + er * d[c];
                    at(V, n, r, c) -= s;
                }
            }
            __syncthreads();
            for (int64_t j = tid; j < i; j += T) {
                d[j] = at(V, n, i - 1, j);
                at(V, n, i, j) = 0.0;
            }
        }
        __syncthreads();
        if (tid == 0) d[i] = h;
        __syncthreads();
    }

    // ---- accumulate the transformations (sym_eig.cpp:85-104) ----------------
    for (int64_t i = 0; i + 1 < n; ++i) {
        if (tid == 0) {
            at(V, n, n - 1, i) = at(V, n, i, i);
            at(V, n, i, i) = 1.0;
        }
        __syncthreads();
        const double h = d[i + 1];
        if (h != 0.0) {
            for (int64_t k = tid; k <= i; k += T) d[k] = at(V, n, k, i + 1) / h;
            __syncthreads();
            for (int64_t j = tid; j <= i; j += T) {
                double g = 0.0;
                for (int64_t k = 0; k <= i; ++k) g += at(V, n, k, i + 1) * at(V, n, k, j);
                for (int64_t k = 0; k <= i; ++k) at(V, n, k, j) -= g * d[k];
            }
            __syncthreads();
        }
        for (int64_t k = tid; k <= i; k += T) at(V, n, k, i + 1) = 0.0;
        __syncthreads();
    }
    for (int64_t j = tid; j < n; j += T) {
        d[j] = at(V, n, n - 1, j);
        at(V, n, n - 1, j) = 0.0;
    }
    __syncthreads();
    if (tid == 0) {
        at(V, n, n - 1, n - 1) = 1.0;
        e[0] = 0.0;
        // ql_implicit's shift of e (sym_eig.cpp:109-110)
        for (int64_t i = 1; i < n; ++i) e[i - 1] = e[i];
        e[n - 1] = 0.0;
    }
    __syncthreads();

    // ---- implicit-shift QL (sym_eig.cpp:107-168) ------------------------------
    // Thread 0 runs the scalar recurrences on (d, e) exactly as the reference
    // and logs each sweep's rotations; every thread then applies them to its
    // rows of V in the reference's order (rotations never depend on V).
    const double eps = 2.220446049250313e-16;
    double f = 0.0, tst1 = 0.0;  // thread 0 only
    for (int64_t l = 0; l < n; ++l) {
        if (tid == 0) {
            tst1 = fmax(tst1, fabs(d[l]) + fabs(e[l]));
            int64_t m = l;
            while (m < n && fabs(e[m]) > eps * tst1) ++m;
            shm[0] = m;
        }
        __syncthreads();
        const int64_t m = shm[0];
        if (m > l) {
            int iter = 0;
            for (;;) {
                if (tid == 0) {
                    flag[0] = 0;
                    if (++iter > kMaxQlSweeps) {
                        flag[0] = 2;
                    } else {
                        double g = d[l];
                        double p = (d[l + 1] - g) / (2.0 * e[l]);
                        double r = hypot(p, 1.0);
                        if (p < 0) r = -r;
                        d[l] = e[l] / (p + r);
                        d[l + 1] = e[l] * (p + r);
                        const double dl1 = d[l + 1];
                        double h = g - d[l];
                        for (int64_t i = l + 2; i < n; ++i) d[i] -= h;
                        f += h;
                        p = d[m];
                        double c = 1.0, c2 = c, c3 = c;
                        const double el1 = e[l + 1];
                        double s = 0.0, s2 = 0.0;
                        for (int64_t i = m; i-- > l;) {
                            c3 = c2;
                            c2 = c;
                            s2 = s;
                            g = c * e[i];
                            h = c * p;
                            r = hypot(p, e[i]);
                            e[i + 1] = s * r;
                            s = e[i] / r;
                            c = p / r;
                            p = c * d[i] - s * g;
                            d[i + 1] = h + s * (c * g + s * d[i]);
                            a.cs[i] = c;
                            a.sn[i] = s;
                        }
                        p = -s * s2 * c3 * el1 * e[l] / dl1;
                        e[l] = s * p;
                        d[l] = c * p;
                        flag[0] = fabs(e[l]) > eps * tst1 ? 1 : 0;
                    }
                }
                __syncthreads();
                const int fl = flag[0];
                if (fl == 2) break;
                for (int64_t k = tid; k < n; k += T) {
                    for (int64_t i = m; i-- > l;) {
                        const double c = a.cs[i], s = a.sn[i];
                        const double h = at(V, n, k, i + 1);
                        at(V, n, k, i + 1) = s * at(V, n, k, i) + c * h;
                        at(V, n, k, i) = c * at(V, n, k, i) - s * h;
                    }
                }
                __syncthreads();
                if (fl == 0) break;
            }
            if (flag[0] == 2) {
                if (tid == 0) a.status[0] = 1;
                return;
            }
        }
        if (tid == 0) {
            d[l] += f;
            e[l] = 0.0;
        }
        __syncthreads();
    }

    // ---- ascending sort carrying the columns (sym_eig.cpp:171-185) -----------
    for (int64_t i = 0; i + 1 < n; ++i) {
        if (tid == 0) {
            int64_t k = i;
            double p = d[i];
            for (int64_t j = i + 1; j < n; ++j)
                if (d[j] < p) {
                    k = j;
                    p = d[j];
                }
            if (k != i) {
                d[k] = d[i];
                d[i] = p;
            }
            shm[1] = k;
        }
        __syncthreads();
        const int64_t k = shm[1];
        if (k != i)
            for (int64_t r = tid; r < n; r += T) {
                const double t = at(V, n, r, i);
                at(V, n, r, i) = at(V, n, r, k);
                at(V, n, r, k) = t;
            }
        __syncthreads();
    }
    if (tid == 0) a.status[0] = 0;
}

// check_symmetric (sym_eig.cpp:13-22): out[0] = max|s|, out[1] = max |s_ij - s_ji|.
__global__ void __launch_bounds__(kDenseThreads) sym_check_kernel(const double* __restrict__ S,
                                                                  int64_t n, double* out) {
    __shared__ double sa[32], sd[32];
    double mx = 0.0, dv = 0.0;
    for (int64_t idx = threadIdx.x; idx < n * n; idx += blockDim.x) {
        const int64_t r = idx % n, c = idx / n;
        mx = fmax(mx, fabs(S[idx]));
        if (r > c) dv = fmax(dv, fabs(S[idx] - S[c + r * n]));
    }
    for (int off = 16; off; off >>= 1) {
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, off));
        dv = fmax(dv, __shfl_xor_sync(0xffffffffu, dv, off));
    }
    if ((threadIdx.x & 31) == 0) {
        sa[threadIdx.x >> 5] = mx;
        sd[threadIdx.x >> 5] = dv;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w) {
            mx = fmax(mx, sa[w]);
            dv = fmax(dv, sd[w]);
        }
        out[0] = mx;
        out[1] = dv;
    }
}

// largest_magnitude_eigenpair's pick and canonical sign (sym_eig.cpp:210-228)
// on the ascending decomposition: out[0] = value, vec = picked column.
__global__ void __launch_bounds__(kDenseThreads) pick_kernel(const double* __restrict__ V,
                                                             const double* __restrict__ w, int64_t n,
                                                             double* __restrict__ out,
                                                             double* __restrict__ vec) {
    __shared__ int64_t sarg;
    const double mlo = fabs(w[0]), mhi = fabs(w[n - 1]);
    const int64_t pick = mlo > mhi * (1.0 + 1e-12) ? 0 : n - 1;
    const double* col = V + pick * n;
    if (threadIdx.x == 0) {
        int64_t arg = 0;
        for (int64_t i = 1; i < n; ++i)
            if (fabs(col[i]) > fabs(col[arg])) arg = i;
        sarg = arg;
        out[0] = w[pick];
    }
    __syncthreads();
    const double sgn = col[sarg] < 0.0 ? -1.0 : 1.0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) vec[i] = sgn < 0.0 ? -col[i] : col[i];
}

// ---- Bunch-Kaufman LDL^T in the reference's storage (sym_eig.cpp:233-320) -----
struct LdltArgs {
    double* W;  // n x n, in: S (lower), out: L below the diagonal, D in the pivot blocks
    int64_t n;
    int* ipiv;
    int* singular;
};

// block-wide (value, index) max with the smallest index on ties
__device__ void argmax_block(double& v, int64_t& idx, double* sv, int64_t* si) {
    for (int off = 16; off; off >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, v, off);
        const int64_t oi = __shfl_xor_sync(0xffffffffu, idx, off);
        if (ov > v || (ov == v && oi < idx)) {
            v = ov;
            idx = oi;
        }
    }
    const int w = threadIdx.x >> 5;
    __syncthreads();
    if ((threadIdx.x & 31) == 0) {
        sv[w] = v;
        si[w] = idx;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int k = 1; k < static_cast<int>(blockDim.x >> 5); ++k)
            if (sv[k] > sv[0] || (sv[k] == sv[0] && si[k] < si[0])) {
                sv[0] = sv[k];
                si[0] = si[k];
            }
    }
    __syncthreads();
    v = sv[0];
    idx = si[0];
}

__global__ void __launch_bounds__(kDenseThreads) ldlt_kernel(LdltArgs a) {
    double* W = a.W;
    const int64_t n = a.n;
    const int tid = threadIdx.x, T = blockDim.x;
    __shared__ double sv[32];
    __shared__ int64_t si[32];
    const double alpha = (1.0 + sqrt(17.0)) / 8.0;
    int sing = 0;
    int64_t k = 0;
    while (k < n) {
        int64_t kstep = 1, kp = k;
        const double absakk = fabs(at(W, n, k, k));
        // colmax / imax: the first row i > k with the largest |w(i, k)| (> 0)
        double cm = 0.0;
        int64_t im = k;
        for (int64_t i = k + 1 + tid; i < n; i += T) {
            const double v = fabs(at(W, n, i, k));
            if (v > cm) {
                cm = v;
                im = i;
            }
        }
        if (cm == 0.0) im = n;  // "no entry beats 0" sorts after every real candidate
        argmax_block(cm, im, sv, si);
        const double colmax = cm;
        const int64_t imax = colmax > 0.0 ? im : k;
        if (fmax(absakk, colmax) == 0.0) {
            sing = 1;
            if (tid == 0) a.ipiv[k] = static_cast<int>(k);
            ++k;
            __syncthreads();
            continue;
        }
        if (absakk >= alpha * colmax) {
            kp = k;
        } else {
            double rm = 0.0;
            for (int64_t j = k + tid; j < imax; j += T) rm = fmax(rm, fabs(at(W, n, imax, j)));
            for (int64_t i = imax + 1 + tid; i < n; i += T) rm = fmax(rm, fabs(at(W, n, i, imax)));
            int64_t dummy = 0;
            argmax_block(rm, dummy, sv, si);
            const double rowmax = rm;
            if (absakk * rowmax >= alpha * colmax * colmax) {
                kp = k;
            } else if (fabs(at(W, n, imax, imax)) >= alpha * rowmax) {
                kp = imax;
            } else {
                kp = imax;
                kstep = 2;
            }
        }
        const int64_t kk = k + kstep - 1;
        if (kp != kk) {
            for (int64_t i = kp + 1 + tid; i < n; i += T) {
                const double t = at(W, n, i, kk);
                at(W, n, i, kk) = at(W, n, i, kp);
                at(W, n, i, kp) = t;
            }
            for (int64_t j = kk + 1 + tid; j < kp; j += T) {
                const double t = at(W, n, j, kk);
                at(W, n, j, kk) = at(W, n, kp, j);
                at(W, n, kp, j) = t;
            }
            if (tid == 0) {
                double t = at(W, n, kk, kk);
                at(W, n, kk, kk) = at(W, n, kp, kp);
                at(W, n, kp, kp) = t;
                if (kstep == 2) {
                    t = at(W, n, k + 1, k);
                    at(W, n, k + 1, k) = at(W, n, kp, k);
                    at(W, n, kp, k) = t;
                }
            }
        }
        __syncthreads();
        if (kstep == 1) {
            const double dkk = at(W, n, k, k);
            if (dkk == 0.0) {
                sing = 1;
            } else {
                const double r1 = 1.0 / dkk;
                for (int64_t j = k + 1; j < n; ++j) {
                    const double cj = r1 * at(W, n, j, k);
                    for (int64_t i = j + tid; i < n; i += T) at(W, n, i, j) -= at(W, n, i, k) * cj;
                }
                __syncthreads();
                for (int64_t i = k + 1 + tid; i < n; i += T) at(W, n, i, k) *= r1;
            }
            if (tid == 0) a.ipiv[k] = static_cast<int>(kp);
        } else {
            if (k + 2 < n) {
                const double d21 = at(W, n, k + 1, k);
                const double d11 = at(W, n, k + 1, k + 1) / d21;
                const double d22 = at(W, n, k, k) / d21;
                const double t = 1.0 / (d11 * d22 - 1.0);
                const double d21t = t / d21;
                for (int64_t j = k + 2; j < n; ++j) {
                    const double wk = d21t * (d11 * at(W, n, j, k) - at(W, n, j, k + 1));
                    const double wkp1 = d21t * (d22 * at(W, n, j, k + 1) - at(W, n, j, k));
                    for (int64_t i = j + tid; i < n; i += T)
                        at(W, n, i, j) -= at(W, n, i, k) * wk + at(W, n, i, k + 1) * wkp1;
                }
                __syncthreads();
                for (int64_t j = k + 2 + tid; j < n; j += T) {
                    const double wk = d21t * (d11 * at(W, n, j, k) - at(W, n, j, k + 1));
                    const double wkp1 = d21t * (d22 * at(W, n, j, k + 1) - at(W, n, j, k));
                    at(W, n, j, k) = wk;
                    at(W, n, j, k + 1) = wkp1;
                }
            }
            if (tid == 0) {
                a.ipiv[k] = -static_cast<int>(kp) - 1;
                a.ipiv[k + 1] = a.ipiv[k];
            }
        }
        k += kstep;
        __syncthreads();
    }
    if (tid == 0) a.singular[0] = sing;
}

// ldlt_solve (sym_eig.cpp:323-377) on the reference storage; b in place.
__global__ void __launch_bounds__(kDenseThreads) ldlt_solve_kernel(const double* __restrict__ W,
                                                                   const int* __restrict__ ipiv,
                                                                   int64_t n, double* b) {
    const int tid = threadIdx.x, T = blockDim.x;
    int64_t k = 0;
    while (k < n) {
        if (ipiv[k] >= 0) {
            const int64_t kp = ipiv[k];
            if (tid == 0 && kp != k) {
                const double t = b[k];
                b[k] = b[kp];
                b[kp] = t;
            }
            __syncthreads();
            const double bk = b[k];
            for (int64_t i = k + 1 + tid; i < n; i += T) b[i] -= at(const_cast<double*>(W), n, i, k) * bk;
            __syncthreads();
            if (tid == 0) b[k] /= W[k + k * n];
            __syncthreads();
            ++k;
        } else {
            const int64_t kp = -ipiv[k] - 1;
            if (tid == 0 && kp != k + 1) {
                const double t = b[k + 1];
                b[k + 1] = b[kp];
                b[kp] = t;
            }
            __syncthreads();
            const double b0 = b[k], b1 = b[k + 1];
            for (int64_t i = k + 2 + tid; i < n; i += T)
                b[i] -= W[i + k * n] * b0 + W[i + (k + 1) * n] * b1;
            __syncthreads();
            if (tid == 0) {
                const double akm1k = W[(k + 1) + k * n];
                const double akm1 = W[k + k * n] / akm1k;
                const double ak = W[(k + 1) + (k + 1) * n] / akm1k;
                const double denom = akm1 * ak - 1.0;
                const double bkm1 = b[k] / akm1k;
                const double bkk = b[k + 1] / akm1k;
                b[k] = (ak * bkm1 - bkk) / denom;
                b[k + 1] = (akm1 * bkk - bkm1) / denom;
            }
            __syncthreads();
            k += 2;
        }
    }
    // backward: the dot products are sequential sums (thread 0, reference order)
    if (tid != 0) return;
    int64_t kb = n;
    while (kb > 0) {
        const int64_t kk = kb - 1;
        if (ipiv[kk] >= 0) {
            double acc = 0.0;
            for (int64_t i = kk + 1; i < n; ++i) acc += W[i + kk * n] * b[i];
            b[kk] -= acc;
            const int64_t kp = ipiv[kk];
            if (kp != kk) {
                const double t = b[kk];
                b[kk] = b[kp];
                b[kp] = t;
            }
            --kb;
        } else {
            double acc0 = 0.0, acc1 = 0.0;
            for (int64_t i = kk + 1; i < n; ++i) {
                acc1 += W[i + kk * n] * b[i];
                acc0 += W[i + (kk - 1) * n] * b[i];
            }
            b[kk] -= acc1;
            b[kk - 1] -= acc0;
            const int64_t kp = -ipiv[kk] - 1;
            if (kp != kk) {
                const double t = b[kk];
                b[kk] = b[kp];
                b[kp] = t;
            }
            kb -= 2;
        }
    }
}

// ldlt_diag_condition (sym_eig.cpp:380-407) from the pivot blocks:
// diag[k] = w(k,k), sub[k] = w(k+1,k) (used at 2x2 starts).
__global__ void diag_cond_kernel(const double* __restrict__ diag, const double* __restrict__ sub,
                                 const int* __restrict__ ipiv, int64_t n, int singular,
                                 double* out) {
    if (threadIdx.x != 0) return;
    if (singular) {
        out[0] = INFINITY;
        return;
    }
    double lo = INFINITY, hi = 0.0;
    int64_t k = 0;
    while (k < n) {
        if (ipiv[k] >= 0) {
            const double m = fabs(diag[k]);
            lo = fmin(lo, m);
            hi = fmax(hi, m);
            ++k;
        } else {
            const double a = diag[k], c = diag[k + 1], bb = sub[k];
            const double mid = 0.5 * (a + c);
            const double rad = hypot(0.5 * (a - c), bb);
            lo = fmin(lo, fmin(fabs(mid + rad), fabs(mid - rad)));
            hi = fmax(hi, fmax(fabs(mid + rad), fabs(mid - rad)));
            k += 2;
        }
    }
    out[0] = lo == 0.0 ? INFINITY : hi / lo;
}

// matricize / dematricize (tensor.cpp:72-98): A viewed as [pre, len, post]
// (first index fastest) <-> M (len x pre*post, column-major), M(i, p + q pre) =
// A[p + pre (i + len q)].
__global__ void unfold_kernel(const double* __restrict__ src, double* __restrict__ dst, int64_t pre,
                              int64_t len, int64_t post, int inverse) {
    const int64_t total = pre * len * post;
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        // t enumerates the tensor (coalesced side)
        const int64_t p = t % pre;
        const int64_t i = (t / pre) % len;
        const int64_t q = t / (pre * len);
        const int64_t m = i + len * (p + q * pre);
        if (inverse)
            dst[t] = src[m];
        else
            dst[m] = src[t];
    }
}

// ttv (tensor.cpp:100-138): A viewed as [pre, len, post]; out[p + pre q] =
// sum_i A[p + pre (i + len q)] v[i], i ascending (the reference's axpy order,
// and its plain dot when pre == 1).
__global__ void ttv_kernel(const double* __restrict__ src, const double* __restrict__ v,
                           double* __restrict__ dst, int64_t pre, int64_t len, int64_t post) {
    const int64_t total = pre * post;
    for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < total;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t p = t % pre, q = t / pre;
        const double* base = src + p + pre * len * q;
        double acc = 0.0;
        for (int64_t i = 0; i < len; ++i) acc += base[pre * i] * v[i];
        dst[t] = acc;
    }
}

// dot (matrix.cpp) of the order-1 remainder with the last vector, sequential.
__global__ void dot_seq_kernel(const double* __restrict__ a, const double* __restrict__ b, int64_t n,
                               double* out) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += a[i] * b[i];
    out[0] = s;
}

// Full decomposition into device buffers: values (n) then vectors (n x n).
void sym_eig_device(r1_context* ctx, int64_t n, const double* s_host, double* ws) {
    double* V = ws + 4 * n + 8;
    double* d = ws;
    double* e = ws + n;
    double* chk = ws + 4 * n;
    int* status = reinterpret_cast<int*>(ws + 4 * n + 4);
    R1_CUDA(cudaMemcpyAsync(V, s_host, static_cast<size_t>(n) * n * sizeof(double),
                            cudaMemcpyHostToDevice, ctx->stream));
    sym_check_kernel<<<1, kDenseThreads, 0, ctx->stream>>>(V, n, chk);
    check_launch(ctx, "sym_check_kernel");
    double h[2];
    R1_CUDA(cudaMemcpyAsync(h, chk, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
    R1_CUDA(cudaStreamSynchronize(ctx->stream));
    if (h[1] > 1e-10 * std::max(h[0], 1e-300))
        fail(R1_ERR_INVALID_ARGUMENT, "sym_eig: matrix is not symmetric");
    if (n == 1) {
        // sym_eig.cpp:196-200
        const double one = 1.0;
        R1_CUDA(cudaMemcpyAsync(d, V, sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
        R1_CUDA(cudaMemcpyAsync(V, &one, sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
        R1_CUDA(cudaStreamSynchronize(ctx->stream));
        return;
    }
    SymEigArgs a{V, d, e, ws + 2 * n, ws + 3 * n, n, status};
    sym_eig_kernel<<<1, kDenseThreads, 0, ctx->stream>>>(a);
    check_launch(ctx, "sym_eig_kernel");
    int st = 0;
    R1_CUDA(cudaMemcpyAsync(&st, status, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    R1_CUDA(cudaStreamSynchronize(ctx->stream));
    if (st != 0) fail(R1_ERR_RUNTIME, "sym_eig: QL iteration did not converge");
}

size_t sym_eig_ws_doubles(int64_t n) { return static_cast<size_t>(n) * n + 4 * n + 16; }

}  // namespace

// largest_magnitude_eigenpair (sym_eig.cpp:206-229) of a DEVICE dense matrix
// S (n x n, overwritten) with the reference's own algorithm, asynchronous:
// value_dev[0], vec_dev[0..n).  ws: 4n + 16 doubles.  (Used by the solvers'
// eigen step for small operators when selected; non-convergence of QL leaves
// the status word in ws[4n+4] nonzero.)
void eig_dense_reference_device(r1_context* ctx, int64_t n, double* S, double* ws, double* value_dev,
                                double* vec_dev) {
    int* status = reinterpret_cast<int*>(ws + 4 * n + 4);
    SymEigArgs a{S, ws, ws + n, ws + 2 * n, ws + 3 * n, n, status};
    sym_eig_kernel<<<1, kDenseThreads, 0, ctx->stream>>>(a);
    check_launch(ctx, "sym_eig_kernel");
    pick_kernel<<<1, kDenseThreads, 0, ctx->stream>>>(S, ws, n, value_dev, vec_dev);
    check_launch(ctx, "pick_kernel");
}

}  // namespace r1

using namespace r1;

extern "C" {

int r1_sym_eig_full(r1_context* ctx, int64_t n, const double* s_host, double* values,
                    double* vectors) {
    return abi_guard([&] {
        CtxLock lk_(ctx);
        if (!ctx) fail(R1_ERR_INVALID_ARGUMENT, "null context");
        R1_CUDA(cudaSetDevice(ctx->device));
        if (n < 0) fail(R1_ERR_INVALID_ARGUMENT, "sym_eig: matrix must be square");
        if (n == 0) return;
        ctx->ws_io.ensure(sym_eig_ws_doubles(n) * sizeof(double));
        double* ws = ctx->ws_io.as<double>();
        sym_eig_device(ctx, n, s_host, ws);
        R1_CUDA(cudaMemcpyAsync(values, ws, n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        R1_CUDA(cudaMemcpyAsync(vectors, ws + 4 * n + 8, static_cast<size_t>(n) * n * sizeof(double),
                                cudaMemcpyDeviceToHost, ctx->stream));
        R1_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

// largest_magnitude_eigenpair (sym_eig.cpp:206-229): the reference's
// definition on the device decomposition.
int r1_largest_magnitude_eigenpair(r1_context* ctx, int64_t n, const double* s_host, double* value,
                                   double* vec) {
    return abi_guard([&] {
        CtxLock lk_(ctx);
        if (!ctx) fail(R1_ERR_INVALID_ARGUMENT, "null context");
        R1_CUDA(cudaSetDevice(ctx->device));
        if (n <= 0) fail(R1_ERR_INVALID_ARGUMENT, "largest_magnitude_eigenpair: empty matrix");
        ctx->ws_io.ensure((sym_eig_ws_doubles(n) + n + 8) * sizeof(double));
        double* ws = ctx->ws_io.as<double>();
        sym_eig_device(ctx, n, s_host, ws);
        double* out = ws + sym_eig_ws_doubles(n);
        pick_kernel<<<1, kDenseThreads, 0, ctx->stream>>>(ws + 4 * n + 8, ws, n, out, out + 8);
        check_launch(ctx, "pick_kernel");
        R1_CUDA(cudaMemcpyAsync(value, out, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        R1_CUDA(cudaMemcpyAsync(vec, out + 8, n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        R1_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

int r1_ldlt_factor(r1_context* ctx, int64_t n, const double* s_host, double* w_host, int* ipiv,
                   int* singular) {
    return abi_guard([&] {
        CtxLock lk_(ctx);
        if (!ctx) fail(R1_ERR_INVALID_ARGUMENT, "null context");
        R1_CUDA(cudaSetDevice(ctx->device));
        if (n < 0) fail(R1_ERR_INVALID_ARGUMENT, "ldlt_factor: matrix must be square");
        *singular = 0;
        if (n == 0) return;
        const size_t nn = static_cast<size_t>(n) * n;
        ctx->ws_io.ensure((nn + n + 16) * sizeof(double));
        double* W = ctx->ws_io.as<double>();
        int* dipiv = reinterpret_cast<int*>(W + nn);
        int* dsing = reinterpret_cast<int*>(W + nn + n + 8);
        R1_CUDA(cudaMemcpyAsync(W, s_host, nn * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
        ldlt_kernel<<<1, kDenseThreads, 0, ctx->stream>>>(LdltArgs{W, n, dipiv, dsing});
        check_launch(ctx, "ldlt_kernel");
        R1_CUDA(cudaMemcpyAsync(w_host, W, nn * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        R1_CUDA(cudaMemcpyAsync(ipiv, dipiv, n * sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
        R1_CUDA(cudaMemcpyAsync(singular, dsing, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
        R1_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

int r1_ldlt_solve(r1_context* ctx, int64_t n, const double* w_host, const int* ipiv,
                  const double* b_host, double* x_host) {
    return abi_guard([&] {
        CtxLock lk_(ctx);
        if (!ctx) fail(R1_ERR_INVALID_ARGUMENT, "null context");
        R1_CUDA(cudaSetDevice(ctx->device));
        if (n <= 0) return;
        const size_t nn = static_cast<size_t>(n) * n;
        ctx->ws_io.ensure((nn + 2 * n + 16) * sizeof(double));
        double* W = ctx->ws_io.as<double>();
        double* b = W + nn;
        int* dipiv = reinterpret_cast<int*>(b + n + 8);
        R1_CUDA(cudaMemcpyAsync(W, w_host, nn * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
        R1_CUDA(cudaMemcpyAsync(b, b_host, n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
        R1_CUDA(cudaMemcpyAsync(dipiv, ipiv, n * sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
        ldlt_solve_kernel<<<1, kDenseThreads, 0, ctx->stream>>>(W, dipiv, n, b);
        check_launch(ctx, "ldlt_solve_kernel");
        R1_CUDA(cudaMemcpyAsync(x_host, b, n * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        R1_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

// diag / sub: the pivot blocks' diagonal and first subdiagonal of w (2n values)
int r1_ldlt_diag_condition(r1_context* ctx, int64_t n, const double* diag, const double* sub,
                           const int* ipiv, int singular, double* out) {
    return abi_guard([&] {
        CtxLock lk_(ctx);
        if (!ctx) fail(R1_ERR_INVALID_ARGUMENT, "null context");
        R1_CUDA(cudaSetDevice(ctx->device));
        ctx->ws_io.ensure((3 * std::max<int64_t>(n, 1) + 16) * sizeof(double));
        double* dd = ctx->ws_io.as<double>();
        double* ds = dd + n;
        double* dout = ds + n;
        int* dipiv = reinterpret_cast<int*>(dout + 8);
        if (n > 0) {
            R1_CUDA(cudaMemcpyAsync(dd, diag, n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
            R1_CUDA(cudaMemcpyAsync(ds, sub, n * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
            R1_CUDA(cudaMemcpyAsync(dipiv, ipiv, n * sizeof(int), cudaMemcpyHostToDevice, ctx->stream));
        }
        diag_cond_kernel<<<1, 32, 0, ctx->stream>>>(dd, ds, dipiv, n, singular, dout);
        check_launch(ctx, "diag_cond_kernel");
        R1_CUDA(cudaMemcpyAsync(out, dout, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        R1_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

// mode-`mode` unfolding; inverse = 1: dematricize (out has the tensor layout)
int r1_matricize(r1_context* ctx, const double* in_host, const uint64_t* dims, int order, int mode,
                 int inverse, double* out_host) {
    return abi_guard([&] {
        CtxLock lk_(ctx);
        if (!ctx) fail(R1_ERR_INVALID_ARGUMENT, "null context");
        R1_CUDA(cudaSetDevice(ctx->device));
        if (mode < 0 || mode >= order)
            fail(R1_ERR_INVALID_ARGUMENT, inverse ? "dematricize: mode out of range"
                                                  : "matricize: mode out of range");
        int64_t pre = 1, post = 1;
        for (int k = 0; k < mode; ++k) pre *= static_cast<int64_t>(dims[k]);
        for (int k = mode + 1; k < order; ++k) post *= static_cast<int64_t>(dims[k]);
        const int64_t len = static_cast<int64_t>(dims[mode]);
        const int64_t total = pre * len * post;
        if (total == 0) return;
        ctx->ws_io.ensure((2 * total + 16) * sizeof(double));
        double* src = ctx->ws_io.as<double>();
        double* dst = src + total + 8;
        h2d_bytes(ctx, src, in_host, total * sizeof(double));
        const int grid = static_cast<int>(std::min<int64_t>((total + 255) / 256, 8 * ctx->num_sms));
        unfold_kernel<<<grid, 256, 0, ctx->stream>>>(src, dst, pre, len, post, inverse);
        check_launch(ctx, "unfold_kernel");
        R1_CUDA(cudaMemcpyAsync(out_host, dst, total * sizeof(double), cudaMemcpyDeviceToHost,
                                ctx->stream));
        R1_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

// ttvc / ttvc_scalar (tensor.cpp:156-199): contract `nmodes` distinct modes in
// descending mode order (vectors vs_host concatenated in the order of `modes`).
// full = 0: out_host receives the remaining tensor (the caller sized it);
// full = 1: all modes, *scalar_out receives the value.
int r1_ttvc(r1_context* ctx, const double* a_host, const uint64_t* dims, int order,
            const double* vs_host, const int* modes, int nmodes, int full, double* out_host,
            double* scalar_out) {
    return abi_guard([&] {
        CtxLock lk_(ctx);
        if (!ctx || !a_host || !dims || (nmodes > 0 && (!vs_host || !modes)))
            fail(R1_ERR_INVALID_ARGUMENT, "null argument");
        R1_CUDA(cudaSetDevice(ctx->device));
        if (order < 1 || order > 16 || nmodes < 1 || nmodes > order)
            fail(R1_ERR_INVALID_ARGUMENT, "ttvc: mode out of range");
        if (full ? nmodes != order : nmodes >= order)
            fail(R1_ERR_INVALID_ARGUMENT, full ? "ttvc_scalar: all modes must be contracted"
                                               : "ttvc: contracting all modes yields a scalar, use ttvc_scalar");
        {
            std::vector<bool> seen(order, false);
            for (int i = 0; i < nmodes; ++i) {
                if (modes[i] < 0 || modes[i] >= order) fail(R1_ERR_INVALID_ARGUMENT, "ttvc: mode out of range");
                if (seen[modes[i]]) fail(R1_ERR_INVALID_ARGUMENT, "ttvc: duplicate mode");
                seen[modes[i]] = true;
            }
        }
        // vector offsets in the caller's order, then the descending contraction order
        std::vector<int64_t> voff(nmodes + 1, 0);
        for (int i = 0; i < nmodes; ++i) voff[i + 1] = voff[i] + static_cast<int64_t>(dims[modes[i]]);
        std::vector<int> ord(nmodes);
        for (int i = 0; i < nmodes; ++i) ord[i] = i;
        std::sort(ord.begin(), ord.end(), [&](int x, int y) { return modes[x] > modes[y]; });
        const r1_tensor* t = upload_tensor(ctx, a_host, dims, order);
        const int64_t numel = static_cast<int64_t>(t->numel);
        const int64_t first_out = numel / static_cast<int64_t>(dims[modes[ord[0]]]);
        const int64_t nv = voff[nmodes];
        ctx->ws_io.ensure((2 * first_out + nv + 64) * sizeof(double));
        double* buf0 = ctx->ws_io.as<double>();
        double* buf1 = buf0 + first_out + 8;
        double* vv = buf1 + first_out + 8;
        double* sc = vv + nv + 8;
        R1_CUDA(cudaMemcpyAsync(vv, vs_host, nv * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
        std::vector<int64_t> cur(dims, dims + order);
        const double* src = t->dev;
        double* dst = buf0;
        const int steps = full ? nmodes - 1 : nmodes;
        for (int s = 0; s < steps; ++s) {
            const int i = ord[s];
            const int mode = modes[i];
            int64_t pre = 1, post = 1;
            for (int k = 0; k < mode; ++k) pre *= cur[k];
            for (size_t k = mode + 1; k < cur.size(); ++k) post *= cur[k];
            const int64_t len = cur[mode];
            const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((pre * post + 255) / 256,
                                                                                    8 * ctx->num_sms)));
            ttv_kernel<<<grid, 256, 0, ctx->stream>>>(src, vv + voff[i], dst, pre, len, post);
            check_launch(ctx, "ttv_kernel");
            cur.erase(cur.begin() + mode);
            src = dst;
            dst = dst == buf0 ? buf1 : buf0;
        }
        int64_t rem = 1;
        for (auto v : cur) rem *= v;
        if (full) {
            const int i = ord[nmodes - 1];
            dot_seq_kernel<<<1, 32, 0, ctx->stream>>>(src, vv + voff[i], rem, sc);
            check_launch(ctx, "dot_seq_kernel");
            R1_CUDA(cudaMemcpyAsync(scalar_out, sc, sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
        } else {
            R1_CUDA(cudaMemcpyAsync(out_host, src, rem * sizeof(double), cudaMemcpyDeviceToHost,
                                    ctx->stream));
        }
        R1_CUDA(cudaStreamSynchronize(ctx->stream));
    });
}

}  // extern "C"
